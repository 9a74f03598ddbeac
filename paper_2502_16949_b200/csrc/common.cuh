// Shared device helpers for the B200 SparseTransX engine (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#ifndef __CUDACC__
#error "compile with nvcc"
#endif

namespace skg {

constexpr unsigned kFull = 0xffffffffu;

// Sticky device error word (ctx->d_err): [0] = code, [1] = batch, [2] = aux,
// [3] = pending per-batch grad flags. Kernels no-op once [0] != 0, which
// preserves the reference's "nothing is applied after the failing batch".
enum ErrCode : uint32_t {
  kErrNone = 0,
  kErrLossNonFinite = 1,     // training.cpp:135-137
  kErrGradEntity = 2,        // embedding.cpp:173 (entity table)
  kErrGradRelation = 3,      // relation table
  kErrGradProj = 4,          // projections
  kErrGradNormals = 5,       // hyperplane normals
  kErrNormalCollapsed = 6,   // embedding.cpp:185-186
  kErrSamplerOverflow = 7,   // device RNG window exhausted (internal)
};
// Pending-flag bits in d_err[3] raised by the forward, resolved after the loss.
enum : uint32_t { kPendEntity = 1u, kPendRelation = 2u, kPendProj = 4u, kPendNormals = 8u };

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define SKG_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw ::skg::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_) + " at " + \
                             __FILE__ + ":" + std::to_string(__LINE__));                 \
  } while (0)

#define SKG_LAUNCH_CHECK() SKG_CUDA(cudaGetLastError())

__device__ __forceinline__ void stamp_now(unsigned long long* p) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *p = t;
}

// Last-block ticket: a gpu-scope acq_rel add publishes this block's partial
// (written before the add, or by its threads before a barrier) and, in the
// block that draws the last ticket, makes every other block's partial visible
// -- without the two full fences of __threadfence + atomicAdd.
__device__ __forceinline__ unsigned ticket_acq_rel(unsigned* counter) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(counter) : "memory");
  return old;
}

__device__ __forceinline__ bool finite_f(float x) { return fabsf(x) <= 3.402823466e38f; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Lemire nearly-divisionless draw, libstdc++ uniform_int_dist.h _S_nd with
// 128-bit products: returns product >> 64; *reject is set when the draw would
// be retried (low < (2^64 - range) % range).
__device__ __forceinline__ uint64_t lemire_hi(uint64_t g, uint64_t range, bool* reject) {
  const uint64_t lo = g * range;
  const uint64_t hi = __umul64hi(g, range);
  bool rej = false;
  if (lo < range) {
    const uint64_t threshold = (0ull - range) % range;
    rej = lo < threshold;
  }
  *reject = rej;
  return hi;
}

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

inline int bits_for(uint64_t max_value) {  // number of bits to represent values <= max_value
  int b = 0;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b;
}

}  // namespace skg
