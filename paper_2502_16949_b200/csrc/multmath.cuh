// Reference arithmetic of the multiplicative family (DistMult / ComplEx /
// RotatE), shared by the training forward (mult.cu) and ranking (eval.cu).
// Complex numbers are float2 (re, im), the interleaved std::complex<float>
// layout of the reference's complex stores (embedding.hpp:15-31).
#pragma once

#include "common.cuh"
#include "kernels.cuh"

namespace skg {

// std::complex<float> / Eigen packet product order, no FMA:
// re = ar*br - ai*bi, im = ar*bi + ai*br.
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(__fsub_rn(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y)),
                     __fadd_rn(__fmul_rn(a.x, b.y), __fmul_rn(a.y, b.x)));
}
__device__ __forceinline__ float2 conj2(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 one2() { return make_float2(1.f, 0.f); }
__device__ __forceinline__ float2 scale2(float u, float2 a) { return make_float2(__fmul_rn(u, a.x), __fmul_rn(u, a.y)); }
// std::abs(std::complex<float>) = cabsf = glibc hypotf: one rounding of the
// double-precision sqrt(x^2 + y^2) (both squares are exact in double).
__device__ __forceinline__ float cabs_ref(float2 q) {
  const double x = q.x, y = q.y;
  return __double2float_rn(__dsqrt_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y))));
}
__device__ __forceinline__ bool finite2(float2 a) { return finite_f(a.x) && finite_f(a.y); }

// Operands of one incidence row, per coordinate. lo / hi are the entity
// columns in ascending order (canonical CSR, sparse.hpp:110-161).
template <int KIND>
struct Unit;

template <>
struct Unit<kDistMult> {
  using T = float;
  static __device__ __forceinline__ T load(const float* X, int64_t row, int W, int c) {
    return __ldg(X + static_cast<size_t>(row) * W + c);
  }
  // ((1 * x_lo) * x_hi) * x_r, and 1 * x is exact
  static __device__ __forceinline__ float term(T h, T t, T r, bool tail_lo) {
    const T lo = tail_lo ? t : h, hi = tail_lo ? h : t;
    return __fmul_rn(__fmul_rn(lo, hi), r);
  }
};

template <>
struct Unit<kComplEx> {
  using T = float2;
  static __device__ __forceinline__ T load(const float* X, int64_t row, int W, int c) {
    return __ldg(reinterpret_cast<const float2*>(X + static_cast<size_t>(row) * W) + c);
  }
  // Re(((1 * y_lo) * y_hi) * r), y_t = conj(t)
  static __device__ __forceinline__ float term(T h, T t, T r, bool tail_lo) {
    const T yt = conj2(t);
    const T lo = tail_lo ? yt : h, hi = tail_lo ? h : yt;
    return cmul(cmul(cmul(one2(), lo), hi), r).x;
  }
};

template <>
struct Unit<kRotatE> {
  using T = float2;
  static __device__ __forceinline__ T load(const float* X, int64_t row, int W, int c) {
    return __ldg(reinterpret_cast<const float2*>(X + static_cast<size_t>(row) * W) + c);
  }
  // q = ((1 * h) * r) - (0 + t): the selecting entries are h and N + r (h is
  // always the lower column), the tail is the subtracted one.
  static __device__ __forceinline__ T q(T h, T t, T r) {
    const T prod = cmul(cmul(one2(), h), r);
    return make_float2(__fsub_rn(prod.x, __fadd_rn(0.f, t.x)), __fsub_rn(prod.y, __fadd_rn(0.f, t.y)));
  }
  static __device__ __forceinline__ float term(T h, T t, T r, bool) { return cabs_ref(q(h, t, r)); }
};

}  // namespace skg
