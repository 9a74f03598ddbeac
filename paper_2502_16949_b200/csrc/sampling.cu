// Device replicas of the reference random streams (see sampling.cuh).
//
// MT19937-64: 156 threads keep the 312-word state in registers (two words
// each) and advance it one full state per block barrier (see mt_kernel).
//
// std::shuffle (libstdc++ stl_algo.h): Fisher-Yates i = 1..n-1, swap(a[i],
// a[j_i]) with j_i uniform in [0, i]; after an optional leading coin call (n
// even) successive i share one draw x in [0, (i+1)(i+2)): j_i = x / (i+2),
// j_{i+1} = x % (i+2). The j_i are computed in parallel; the permutation is
// then replayed without the sequential swap chain: value v lands at j_v at
// step v and afterwards moves to position i at the first later step whose
// j_i equals its current position. Grouping steps by j (stable radix sort)
// gives those "next step" links, and each value walks its own short chain.
#include "common.cuh"
#include "sampling.cuh"

namespace skg {

namespace {

constexpr uint64_t kMatA = 0xB5026F5AA96619E9ULL;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL;
constexpr uint64_t kLower = 0x000000007FFFFFFFULL;
constexpr int kMtN = 312;
constexpr int kMtM = 156;
constexpr int kShiftWindow = 40;     // max Lemire rejections per shuffle handled in parallel
constexpr int kCandCap = 4096;
constexpr uint32_t kNone = 0xFFFFFFFFu;

__device__ __forceinline__ uint64_t mt_mix(uint64_t a, uint64_t b) {
  const uint64_t y = (a & kUpper) | (b & kLower);
  return (y >> 1) ^ ((y & 1ull) ? kMatA : 0ull);
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

__device__ void mt_seed(uint64_t seed, uint64_t* x) {
  x[0] = seed;
  for (int i = 1; i < kMtN; ++i) x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + i;
}

// Register-resident twist: thread i (< 156) keeps a_i = x[i] and b_i =
// x[156 + i] of the current state. The next state is
//   a'_i = b_i ^ mix(a_i, a_{i+1})            (a_156 := b_0)
//   b'_i = a'_i ^ mix(b_i, b_{i+1})           (i < 155)
//   b'_155 = a'_155 ^ mix(b_155, a'_0)
// so one state needs only the neighbours' previous words: every thread
// publishes (a_i, b_i) to a double-buffered shared array, one barrier per
// state, and thread 155 recomputes a'_0 itself. Tempering and the coalesced
// stores of both halves are off the dependency chain.
constexpr int kMtThreads = 160;

__global__ void __launch_bounds__(kMtThreads) mt_kernel(const uint64_t* __restrict__ seed_ptr,
                                                        uint64_t seed_val, uint64_t* __restrict__ out,
                                                        int64_t n) {
  __shared__ uint64_t sa[2][kMtM + 1], sb[2][kMtM + 1];
  __shared__ uint64_t init[kMtN];
  const int i = threadIdx.x;
  if (i == 0) mt_seed(seed_ptr ? *seed_ptr : seed_val, init);
  __syncthreads();
  const bool on = i < kMtM;
  uint64_t a = on ? init[i] : 0ull, b = on ? init[kMtM + i] : 0ull;
  const int64_t nstates = (n + kMtN - 1) / kMtN;
  int cur = 0;
  for (int64_t s = 0; s < nstates; ++s) {
    if (on) {
      sa[cur][i] = a;
      sb[cur][i] = b;
    }
    __syncthreads();
    if (on) {
      const uint64_t a1 = i + 1 < kMtM ? sa[cur][i + 1] : sb[cur][0];
      const uint64_t na = b ^ mt_mix(a, a1);
      uint64_t nb;
      if (i + 1 < kMtM) {
        nb = na ^ mt_mix(b, sb[cur][i + 1]);
      } else {  // b'_155 needs a'_0 = b_0 ^ mix(a_0, a_1)
        const uint64_t na0 = sb[cur][0] ^ mt_mix(sa[cur][0], sa[cur][1]);
        nb = na ^ mt_mix(b, na0);
      }
      a = na;
      b = nb;
      const int64_t base = s * kMtN;
      if (base + i < n) out[base + i] = mt_temper(a);
      if (base + kMtM + i < n) out[base + kMtM + i] = mt_temper(b);
    }
    cur ^= 1;
  }
}

// Chunked stream: block j generates words [j L, min((j + 1) L, n)) of the
// same stream, starting from the seeded state advanced j L words. The jump
// evaluates sum_i p_i A^i s0 for p = x^(jL) mod f (mt_jump.cpp) by Horner's
// rule 64 coefficients at a time: acc = A^64(acc) ^ sum_k p_(64w+k) A^k s0,
// where A^64 is 64 independent word steps (each new word reads only words of
// the old window) and A^k s0 is s0's own word sequence from word k. L is a
// multiple of 312, so every chunk starts on a whole state and continues with
// the register twist of mt_kernel.
constexpr int kJumpThreads = 320;
constexpr int kJumpWords = 312;  // coefficient words per jump polynomial (19937 bits)

__global__ void __launch_bounds__(kJumpThreads) mt_chunk_kernel(const uint64_t* __restrict__ seed_ptr,
                                                                uint64_t seed_val,
                                                                const uint64_t* __restrict__ polys, int64_t L,
                                                                uint64_t* __restrict__ out, int64_t n) {
  __shared__ uint64_t s0[kMtN + 64];  // seeded state and the next 64 words of its sequence
  __shared__ uint64_t acc[kMtN];
  __shared__ uint64_t sa[2][kMtM + 1], sb[2][kMtM + 1];
  const int tid = threadIdx.x;
  const int64_t j = blockIdx.x;
  if (tid == 0) mt_seed(seed_ptr ? *seed_ptr : seed_val, s0);
  __syncthreads();
  if (tid < 64) s0[kMtN + tid] = s0[kMtM + tid] ^ mt_mix(s0[tid], s0[tid + 1]);
  for (int i = tid; i < kMtN; i += blockDim.x) acc[i] = j == 0 ? s0[i] : 0ull;
  __syncthreads();
  int h = 0;
  if (j > 0) {
    const uint64_t* p = polys + (j - 1) * kJumpWords;
    for (int wi = kJumpWords - 1; wi >= 0; --wi) {
      const uint64_t bits = __ldg(p + wi);  // block-uniform
      // acc = A^64(acc): 64 independent word steps (reads of the old window first)
      uint64_t nw = 0;
      int slot = 0;
      if (tid < 64) {
        int k0 = h + tid;
        k0 -= k0 >= kMtN ? kMtN : 0;
        int k1 = k0 + 1;
        k1 -= k1 >= kMtN ? kMtN : 0;
        int km = k0 + kMtM;
        km -= km >= kMtN ? kMtN : 0;
        nw = acc[km] ^ mt_mix(acc[k0], acc[k1]);
        slot = k0;
      }
      __syncthreads();
      if (tid < 64) acc[slot] = nw;
      h += 64;
      h -= h >= kMtN ? kMtN : 0;
      __syncthreads();
      // acc ^= sum_k p_(64 wi + k) A^k s0: a uniform branch per coefficient,
      // consecutive threads read consecutive words of s0's sequence
      if (bits && tid < kMtN) {
        // four independent XOR chains so the shared-memory loads overlap
        uint64_t x0 = 0, x1 = 0, x2 = 0, x3 = 0;
        const uint64_t* src = s0 + tid;
#pragma unroll
        for (int k = 0; k < 64; k += 4) {
          if ((bits >> k) & 1u) x0 ^= src[k];
          if ((bits >> (k + 1)) & 1u) x1 ^= src[k + 1];
          if ((bits >> (k + 2)) & 1u) x2 ^= src[k + 2];
          if ((bits >> (k + 3)) & 1u) x3 ^= src[k + 3];
        }
        const uint64_t x = (x0 ^ x1) ^ (x2 ^ x3);
        int w = h + tid;
        w -= w >= kMtN ? kMtN : 0;
        acc[w] ^= x;
      }
      __syncthreads();
    }
  }
  // generate the chunk from the jumped window (thread i < 156 keeps words i and 156 + i)
  const bool on = tid < kMtM;
  int ia = h + tid, ib = h + kMtM + tid;
  ia -= ia >= kMtN ? kMtN : 0;
  ib -= ib >= kMtN ? kMtN : 0;
  ib -= ib >= kMtN ? kMtN : 0;
  uint64_t a = on ? acc[ia] : 0ull, b = on ? acc[ib] : 0ull;
  const int64_t w0 = j * L, w1 = min(n, w0 + L);
  const int64_t nstates = (w1 - w0 + kMtN - 1) / kMtN;
  int cur = 0;
  for (int64_t st = 0; st < nstates; ++st) {
    if (on) {
      sa[cur][tid] = a;
      sb[cur][tid] = b;
    }
    __syncthreads();
    if (on) {
      const uint64_t a1 = tid + 1 < kMtM ? sa[cur][tid + 1] : sb[cur][0];
      const uint64_t na = b ^ mt_mix(a, a1);
      uint64_t nb;
      if (tid + 1 < kMtM) {
        nb = na ^ mt_mix(b, sb[cur][tid + 1]);
      } else {
        const uint64_t na0 = sb[cur][0] ^ mt_mix(sa[cur][0], sa[cur][1]);
        nb = na ^ mt_mix(b, na0);
      }
      a = na;
      b = nb;
      const int64_t base = w0 + st * kMtN;
      if (base + tid < w1) out[base + tid] = mt_temper(a);
      if (base + kMtM + tid < w1) out[base + kMtM + tid] = mt_temper(b);
    }
    cur ^= 1;
  }
}

// Sequential single-thread MT19937-64 (fallback paths only).
struct SeqMt {
  uint64_t x[kMtN];
  int p;
  __device__ void init(uint64_t seed) {
    mt_seed(seed, x);
    p = kMtN;
  }
  __device__ uint64_t next() {
    if (p >= kMtN) {
      for (int k = 0; k < kMtN - kMtM; ++k) x[k] = x[k + kMtM] ^ mt_mix(x[k], x[k + 1]);
      for (int k = kMtN - kMtM; k < kMtN - 1; ++k) x[k] = x[k - (kMtN - kMtM)] ^ mt_mix(x[k], x[k + 1]);
      x[kMtN - 1] = x[kMtM - 1] ^ mt_mix(x[kMtN - 1], x[0]);
      p = 0;
    }
    return mt_temper(x[p++]);
  }
  __device__ uint64_t uniform(uint64_t range) {  // _S_nd with retries
    bool rej;
    uint64_t hi;
    do {
      hi = lemire_hi(next(), range, &rej);
    } while (rej);
    return hi;
  }
};

// ---------------------------------------------------------------- shuffle

struct CallInfo {
  int64_t i;       // first swap index of this call
  uint64_t range;  // Lemire range
  bool coin;
};

__device__ __forceinline__ CallInfo call_info(int64_t c, int64_t n) {
  CallInfo ci;
  if ((n & 1) == 0) {
    if (c == 0) {
      ci.i = 1;
      ci.range = 2;
      ci.coin = true;
      return ci;
    }
    ci.i = 2 * c;
  } else {
    ci.i = 2 * c + 1;
  }
  ci.range = static_cast<uint64_t>(ci.i + 1) * static_cast<uint64_t>(ci.i + 2);
  ci.coin = false;
  return ci;
}

__host__ __device__ __forceinline__ int64_t num_calls(int64_t n) {
  if (n <= 1) return 0;
  return (n & 1) == 0 ? 1 + (n - 2) / 2 : (n - 1) / 2;
}

__global__ void shuffle_reset_kernel(uint32_t* ncand, uint32_t* nshift) {
  ncand[0] = 0;
  ncand[1] = 0;
  *nshift = 0;
}

__global__ void shuffle_candidates_kernel(const uint64_t* __restrict__ raw, int64_t nraw, int64_t n,
                                          uint64_t* __restrict__ cand, uint32_t* __restrict__ ncand) {
  const int64_t C = num_calls(n);
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < C;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const CallInfo ci = call_info(c, n);
    if (ci.coin) continue;  // range 2 never rejects: (2^64 - 2) % 2 == 0
#pragma unroll 4
    for (int s = 0; s < kShiftWindow; ++s) {
      const int64_t q = c + s;
      if (q >= nraw) break;
      bool rej;
      lemire_hi(raw[q], ci.range, &rej);
      if (rej) {
        const uint32_t k = atomicAdd(&ncand[0], 1u);
        if (k < kCandCap)
          cand[k] = (static_cast<uint64_t>(c) << 8) | static_cast<uint64_t>(s);
        else
          ncand[1] = 1;
      }
    }
  }
}

// One CTA: sort candidates, then walk them in call order to get the exact
// shift (extra draws consumed so far) in force from each rejecting call on.
__global__ void __launch_bounds__(1024) shuffle_resolve_kernel(const uint64_t* __restrict__ cand,
                                                               uint32_t* __restrict__ ncand,
                                                               uint64_t* __restrict__ shifts,
                                                               uint32_t* __restrict__ nshift) {
  __shared__ uint64_t sk[kCandCap];
  const uint32_t k = min(ncand[0], static_cast<uint32_t>(kCandCap));
  if (k == 0) return;
  int p2 = 1;
  while (p2 < static_cast<int>(k)) p2 <<= 1;
  for (int t = threadIdx.x; t < p2; t += blockDim.x) sk[t] = t < static_cast<int>(k) ? cand[t] : ~0ull;
  __syncthreads();
  for (int size = 2; size <= p2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < p2; t += blockDim.x) {
        const int o = t ^ stride;
        if (o > t) {
          const bool up = (t & size) == 0;
          const uint64_t a = sk[t], b = sk[o];
          if ((a > b) == up) {
            sk[t] = b;
            sk[o] = a;
          }
        }
      }
      __syncthreads();
    }
  if (threadIdx.x == 0) {
    uint32_t shift = 0, ns = 0;
    int64_t cur_c = -1;
    uint32_t shift_at_start = 0;
    for (uint32_t t = 0; t < k; ++t) {
      const int64_t c = static_cast<int64_t>(sk[t] >> 8);
      const uint32_t s = static_cast<uint32_t>(sk[t] & 0xff);
      if (c != cur_c) {
        if (cur_c >= 0 && shift != shift_at_start) shifts[ns++] = (static_cast<uint64_t>(cur_c) << 8) | shift;
        cur_c = c;
        shift_at_start = shift;
      }
      if (s == shift) ++shift;
    }
    if (cur_c >= 0 && shift != shift_at_start) shifts[ns++] = (static_cast<uint64_t>(cur_c) << 8) | shift;
    if (shift >= static_cast<uint32_t>(kShiftWindow)) ncand[1] = 1;
    *nshift = ns;
  }
}

__global__ void shuffle_map_kernel(const uint64_t* __restrict__ raw, int64_t n,
                                   const uint64_t* __restrict__ shifts,
                                   const uint32_t* __restrict__ nshift, uint32_t* __restrict__ jpos) {
  const int64_t C = num_calls(n);
  const uint32_t ns = *nshift;
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < C;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // last table entry with call <= c
    uint32_t lo = 0, hi = ns, shift = 0;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (static_cast<int64_t>(shifts[mid] >> 8) <= c)
        lo = mid + 1;
      else
        hi = mid;
    }
    if (lo > 0) shift = static_cast<uint32_t>(shifts[lo - 1] & 0xff);
    const CallInfo ci = call_info(c, n);
    bool rej;
    const uint64_t x = lemire_hi(raw[c + shift], ci.range, &rej);
    if (ci.coin) {
      jpos[1] = static_cast<uint32_t>(x);
    } else {
      const uint64_t b1 = static_cast<uint64_t>(ci.i + 2);
      jpos[ci.i] = static_cast<uint32_t>(x / b1);
      jpos[ci.i + 1] = static_cast<uint32_t>(x % b1);
    }
  }
}

// Exact sequential std::shuffle; only runs when the parallel window overflowed.
__global__ void shuffle_fallback_kernel(const uint64_t* __restrict__ seed_ptr, int64_t n,
                                        int32_t* __restrict__ order, const uint32_t* __restrict__ ncand) {
  if (ncand[1] == 0) return;
  SeqMt g;
  g.init(*seed_ptr);
  for (int64_t i = 0; i < n; ++i) order[i] = static_cast<int32_t>(i);
  if (n <= 1) return;
  int64_t i = 1;
  if ((n & 1) == 0) {
    const int64_t j = static_cast<int64_t>(g.uniform(2));
    const int32_t t = order[i];
    order[i] = order[j];
    order[j] = t;
    ++i;
  }
  while (i < n) {
    const uint64_t b1 = static_cast<uint64_t>(i + 2);
    const uint64_t x = g.uniform(static_cast<uint64_t>(i + 1) * b1);
    const int64_t j0 = static_cast<int64_t>(x / b1), j1 = static_cast<int64_t>(x % b1);
    int32_t t = order[i];
    order[i] = order[j0];
    order[j0] = t;
    ++i;
    t = order[i];
    order[i] = order[j1];
    order[j1] = t;
    ++i;
  }
}

__global__ void shuffle_keys_kernel(const uint32_t* __restrict__ jpos, int64_t n,
                                    uint32_t* __restrict__ key, uint32_t* __restrict__ val) {
  for (int64_t i = 1 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    key[i - 1] = jpos[i];
    val[i - 1] = static_cast<uint32_t>(i);
  }
}

__global__ void shuffle_groups_kernel(const uint32_t* __restrict__ key, const uint32_t* __restrict__ val,
                                      int64_t cnt, uint32_t* __restrict__ gstart,
                                      uint32_t* __restrict__ nextsame) {
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < cnt;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t k = key[q];
    if (q == 0 || key[q - 1] != k) gstart[k] = static_cast<uint32_t>(q);
    nextsame[val[q]] = (q + 1 < cnt && key[q + 1] == k) ? val[q + 1] : kNone;
  }
}

__device__ __forceinline__ uint32_t first_after(uint32_t k, const uint32_t* gstart, const uint32_t* val,
                                                const uint32_t* nextsame) {
  const uint32_t g = gstart[k];
  if (g == kNone) return kNone;
  const uint32_t i0 = val[g];
  return i0 != k ? i0 : nextsame[i0];
}

__global__ void shuffle_walk_kernel(const uint32_t* __restrict__ jpos, int64_t n,
                                    const uint32_t* __restrict__ gstart, const uint32_t* __restrict__ val,
                                    const uint32_t* __restrict__ nextsame, int32_t* __restrict__ order,
                                    const uint32_t* __restrict__ ncand) {
  if (ncand[1] != 0) return;  // fallback produced the order
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t pos, nxt;
    if (v == 0) {
      pos = 0;
      nxt = n > 1 ? first_after(0, gstart, val, nextsame) : kNone;
    } else {
      pos = jpos[v];
      nxt = nextsame[v];
    }
    while (nxt != kNone) {
      pos = nxt;
      nxt = first_after(nxt, gstart, val, nextsame);
    }
    order[pos] = static_cast<int32_t>(v);
  }
}

__global__ void iota_kernel(int32_t* __restrict__ order, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    order[i] = static_cast<int32_t>(i);
}

// ---------------------------------------------------------------- negatives

// draw_excluding (training.cpp:22-31) for one triple given its two raw draws
__device__ __forceinline__ int32_t corrupt_one(uint64_t g, int32_t orig, int32_t other, int64_t n,
                                               bool avoid, bool* reject) {
  const int64_t ex1 = avoid ? other : orig;
  const int64_t lo = min(static_cast<int64_t>(orig), ex1), hi = max(static_cast<int64_t>(orig), ex1);
  const int64_t k = lo == hi ? 1 : 2;
  const uint64_t range = static_cast<uint64_t>(n - k);
  int64_t v = static_cast<int64_t>(lemire_hi(g, range, reject));
  if (v >= lo) ++v;
  if (k == 2 && v >= hi) ++v;
  return static_cast<int32_t>(v);
}

__global__ void neg_map_kernel(const uint64_t* __restrict__ raw, const int32_t* __restrict__ h,
                               const int32_t* __restrict__ t, int64_t m, int64_t n, int avoid,
                               int32_t* __restrict__ oh, int32_t* __restrict__ ot,
                               uint32_t* __restrict__ first_reject) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const bool corrupt_head = (raw[2 * i] >> 63) == 0;  // coin(0,1) == 0: top bit of the draw
    const int32_t hh = h[i], tt = t[i];
    bool rej;
    const int32_t v = corrupt_one(raw[2 * i + 1], corrupt_head ? hh : tt, corrupt_head ? tt : hh, n,
                                  avoid != 0, &rej);
    if (rej) atomicMin(first_reject, static_cast<uint32_t>(i));
    oh[i] = corrupt_head ? v : hh;
    ot[i] = corrupt_head ? tt : v;
  }
}

// Sequential continuation from the first rejecting triple (probability ~1e-13
// per draw); consumes the raw stream exactly like the reference loop.
__global__ void neg_fixup_kernel(const uint64_t* __restrict__ raw, int64_t nraw,
                                 const int32_t* __restrict__ h, const int32_t* __restrict__ t,
                                 int64_t m, int64_t n, int avoid, int32_t* __restrict__ oh,
                                 int32_t* __restrict__ ot, uint32_t* __restrict__ first_reject) {
  const uint32_t f = *first_reject;
  if (f == kNone) return;
  int64_t q = 2 * static_cast<int64_t>(f);
  for (int64_t i = f; i < m; ++i) {
    if (q + 2 > nraw) {
      first_reject[1] = 1;  // window exhausted
      return;
    }
    const bool corrupt_head = (raw[q++] >> 63) == 0;
    const int32_t hh = h[i], tt = t[i];
    int32_t v;
    bool rej;
    do {
      if (q >= nraw) {
        first_reject[1] = 1;
        return;
      }
      v = corrupt_one(raw[q++], corrupt_head ? hh : tt, corrupt_head ? tt : hh, n, avoid != 0, &rej);
    } while (rej);
    oh[i] = corrupt_head ? v : hh;
    ot[i] = corrupt_head ? tt : v;
  }
}

int grid_for(int64_t n, int threads = 256) {
  const int64_t b = (n + threads - 1) / threads;
  return static_cast<int>(b < 1 ? 1 : (b > 4096 ? 4096 : b));
}

}  // namespace

// Chunk plan of a raw stream of n words: P chunks of L words (L a multiple of
// 312) with their jump polynomials on device; P = 1 below ~320 K words, where
// the single-block generator is faster than a jump.
void MtJump::prepare(int64_t n) {
  if (n == n_prepared) return;
  int64_t P = n / (static_cast<int64_t>(kMtN) * 1024);
  P = P < 2 ? 1 : (P > 32 ? 32 : P);
  int64_t L = (n + P - 1) / P;
  L = (L + kMtN - 1) / kMtN * kMtN;
  P = (n + L - 1) / L;
  chunks = static_cast<int>(P);
  chunk_words = L;
  if (P > 1) {
    const std::vector<uint64_t>& h = mt_jump_polys(L, static_cast<int>(P));
    if (static_cast<int64_t>(h.size()) > cap) {
      if (polys) cudaFree(polys);
      SKG_CUDA(cudaMalloc(&polys, sizeof(uint64_t) * h.size()));
      cap = static_cast<int64_t>(h.size());
    }
    SKG_CUDA(cudaMemcpy(polys, h.data(), sizeof(uint64_t) * h.size(), cudaMemcpyHostToDevice));
  }
  n_prepared = n;
}

void MtJump::release() {
  if (polys) cudaFree(polys);
  polys = nullptr;
  cap = 0;
  n_prepared = -1;
}

void MtJump::generate(const uint64_t* seed_ptr, uint64_t seed_val, uint64_t* out, int64_t n, cudaStream_t s) const {
  if (n != n_prepared) throw CudaError("mt stream: jump plan not prepared for this length");
  if (chunks <= 1) {
    mt_kernel<<<1, kMtThreads, 0, s>>>(seed_ptr, seed_val, out, n);
  } else {
    mt_chunk_kernel<<<chunks, kJumpThreads, 0, s>>>(seed_ptr, seed_val, polys, chunk_words, out, n);
  }
  count_launch();
  SKG_LAUNCH_CHECK();
}

void mt19937_64_generate(uint64_t seed, uint64_t* out, int64_t n, cudaStream_t s) {
  mt_kernel<<<1, kMtThreads, 0, s>>>(nullptr, seed, out, n);
  count_launch();
  SKG_LAUNCH_CHECK();
}

void ShuffleWork::reserve(int64_t n) {
  // the jump plan follows the current length (prepare_epoch runs this outside any capture)
  if (n <= cap_n) {
    jump.prepare(num_calls(n) + kShiftWindow + 64);
    return;
  }
  release();
  const int64_t nraw = num_calls(n) + kShiftWindow + 64;
  SKG_CUDA(cudaMalloc(&raw, sizeof(uint64_t) * nraw));
  jump.prepare(nraw);  // uploads the jump polynomials
  SKG_CUDA(cudaMalloc(&cand, sizeof(uint64_t) * kCandCap));
  SKG_CUDA(cudaMalloc(&ncand, sizeof(uint32_t) * 2));
  SKG_CUDA(cudaMalloc(&shifts, sizeof(uint64_t) * kCandCap));
  SKG_CUDA(cudaMalloc(&nshift, sizeof(uint32_t)));
  for (uint32_t** p : {&jkey, &jval, &jkey_alt, &jval_alt, &jpos, &gstart, &nextsame})
    SKG_CUDA(cudaMalloc(p, sizeof(uint32_t) * (n + 1)));
  sort.reserve(n);
  cap_n = n;
}

void ShuffleWork::release() {
  for (void* p : {(void*)raw, (void*)cand, (void*)ncand, (void*)shifts, (void*)nshift, (void*)jkey,
                  (void*)jval, (void*)jkey_alt, (void*)jval_alt, (void*)jpos, (void*)gstart,
                  (void*)nextsame})
    if (p) cudaFree(p);
  raw = cand = shifts = nullptr;
  ncand = nshift = jkey = jval = jkey_alt = jval_alt = jpos = gstart = nextsame = nullptr;
  cap_n = 0;
  sort.release();
  jump.release();
}

void device_iota(int32_t* order, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  iota_kernel<<<grid_for(n), 256, 0, s>>>(order, n);
  count_launch();
  SKG_LAUNCH_CHECK();
}

void device_shuffle(const uint64_t* d_seed_eff, int64_t n, int32_t* order, ShuffleWork& w,
                    cudaStream_t s) {
  if (n <= 1) {
    device_iota(order, n, s);
    return;
  }
  w.reserve(n);
  const int64_t C = num_calls(n);
  const int64_t nraw = C + kShiftWindow + 64;
  shuffle_reset_kernel<<<1, 1, 0, s>>>(w.ncand, w.nshift);
  count_launch();
  w.jump.prepare(nraw);  // no-op after reserve (a smaller n than reserved re-plans, never inside a capture)
  w.jump.generate(d_seed_eff, 0, w.raw, nraw, s);
  shuffle_candidates_kernel<<<grid_for(C), 256, 0, s>>>(w.raw, nraw, n, w.cand, w.ncand);
  shuffle_resolve_kernel<<<1, 1024, 0, s>>>(w.cand, w.ncand, w.shifts, w.nshift);
  shuffle_map_kernel<<<grid_for(C), 256, 0, s>>>(w.raw, n, w.shifts, w.nshift, w.jpos);
  shuffle_fallback_kernel<<<1, 1, 0, s>>>(d_seed_eff, n, order, w.ncand);
  shuffle_keys_kernel<<<grid_for(n), 256, 0, s>>>(w.jpos, n, w.jkey, w.jval);
  count_launch(5);
  SKG_LAUNCH_CHECK();
  const int kb = bits_for(static_cast<uint64_t>(n - 1));
  const bool alt = radix_sort_pairs(w.jkey, w.jval, w.jkey_alt, w.jval_alt, n - 1, kb, w.sort, s);
  const uint32_t* sk = alt ? w.jkey_alt : w.jkey;
  const uint32_t* sv = alt ? w.jval_alt : w.jval;
  SKG_CUDA(cudaMemsetAsync(w.gstart, 0xFF, sizeof(uint32_t) * n, s));
  shuffle_groups_kernel<<<grid_for(n), 256, 0, s>>>(sk, sv, n - 1, w.gstart, w.nextsame);
  shuffle_walk_kernel<<<grid_for(n), 256, 0, s>>>(w.jpos, n, w.gstart, sv, w.nextsame, order, w.ncand);
  count_launch(2);
  SKG_LAUNCH_CHECK();
}

void NegWork::reserve(int64_t m) {
  if (m <= cap) return;
  release();
  SKG_CUDA(cudaMalloc(&raw, sizeof(uint64_t) * (2 * m + 4096)));
  SKG_CUDA(cudaMalloc(&first_reject, sizeof(uint32_t) * 2));
  cap = m;
}

void NegWork::release() {
  if (raw) cudaFree(raw);
  if (first_reject) cudaFree(first_reject);
  raw = nullptr;
  first_reject = nullptr;
  cap = 0;
  jump.release();
}

bool device_negative_sample(const int32_t* h, const int32_t* t, int64_t m, int64_t n_ent,
                            uint64_t seed, bool avoid, int32_t* out_h, int32_t* out_t, NegWork& w,
                            cudaStream_t s) {
  if (m <= 0) return true;
  w.reserve(m);
  const int64_t nraw = 2 * m + 4096;
  SKG_CUDA(cudaMemsetAsync(w.first_reject, 0xFF, sizeof(uint32_t), s));
  SKG_CUDA(cudaMemsetAsync(w.first_reject + 1, 0, sizeof(uint32_t), s));
  w.jump.prepare(nraw);  // eager path (never captured)
  w.jump.generate(nullptr, seed, w.raw, nraw, s);
  neg_map_kernel<<<grid_for(m), 256, 0, s>>>(w.raw, h, t, m, n_ent, avoid ? 1 : 0, out_h, out_t,
                                             w.first_reject);
  neg_fixup_kernel<<<1, 1, 0, s>>>(w.raw, nraw, h, t, m, n_ent, avoid ? 1 : 0, out_h, out_t,
                                   w.first_reject);
  count_launch(2);
  SKG_LAUNCH_CHECK();
  uint32_t flags[2];
  SKG_CUDA(cudaMemcpyAsync(flags, w.first_reject, sizeof(flags), cudaMemcpyDeviceToHost, s));
  SKG_CUDA(cudaStreamSynchronize(s));
  return flags[1] == 0;
}

}  // namespace skg
