// Row-sharded data parallel for the hrt models (TransE / TorusE; SURVEY §8e,
// the wikikg2-scale layout BASELINE.json's north_star asks for).
//
// G ranks (G = 1, 2, 4 or 8), one GPU each. Every global minibatch of the
// reference trainer (training.cpp:120-161 at batch_size = global batch) is
// split into G contiguous pair shards, rank k computing the forward of shard
// k. The parameters are split by OWNER instead of being replicated:
//   - entity e lives only on rank e % G, at local row e / G;
//   - the relation table (R x d, 0.5 MB for wikikg2) is replicated, and
//     relation r is reduced and updated by rank r % G, which then writes the
//     new row into every rank's replica.
// Per batch:
//   1. forward (hrt_forward_kernel, SH = true): each rank gathers its pairs'
//      entity rows straight from the owners' shards over NVLink (peer loads)
//      and its relation rows from the local replica; residual rows and row
//      scales stay in the rank's own HBM;
//   2. barrier;
//   3. backward (shard_segment_kernel): each rank reduces the columns it owns.
//      Its plan lists, for the whole GLOBAL batch, only the incidence entries
//      of owned columns, in the reference's accumulation order (positive rows
//      ascending, then negative rows ascending; sparse.hpp:268-272,
//      training.cpp:146-147) -- the same stable (batch, column) sort as the
//      single-GPU plan -- so every sum is bitwise the reference's at
//      batch_size = G x shard. Residual rows are pulled from the rank that
//      computed them (peer loads). SGD is applied in place (entities) or
//      broadcast to every replica (relations);
//   4. barrier.
// Bytes moved over NVLink per batch (rank view, d floats per row, B global
// pairs): forward ~ (G-1)/G x 4B x d x 4 entity-row reads; backward
// ~ (G-1)/G x (#entries it owns) x d x 4 residual-row reads + (G-1) x
// (owned relation rows) x d x 4 replica writes. No parameter table is ever
// reduced densely: what crosses the links is proportional to the batch, not to
// the table (2.56 GB for wikikg2), which the replicated design all-reduced
// every batch.
//
// Barrier: a one-block kernel per rank in the captured epoch graph. Rank g
// writes its generation (and its sticky error code) into slot g of every
// rank's flag array with a system-scope release store and spins on its own
// array with acquire loads; a non-finite loss on any shard therefore stops
// every rank at the same batch (the global loss is non-finite iff a shard's
// is). A 20 s timeout turns a lost peer into an error instead of a hang.
//
// Peer pointers come either from another context of the same process
// (skg_shard_group_init: one process driving all ranks, or G contexts on one
// GPU for the tests) or from CUDA IPC handles exchanged by the caller
// (skg_shard_export / skg_shard_import: one process per GPU). The sharded
// buffers live in one cudaMalloc arena so one handle covers them.
#include <cstring>

#include "common.cuh"
#include "engine.cuh"
#include "ht.cuh"
#include "kernels.cuh"
#include "plan.cuh"
#include "primitives.cuh"
#include "refmath.cuh"
#include "shard.cuh"

namespace skg {

namespace {

constexpr uint32_t kRelFlag = 0x80000000u;  // seg_col of a relation segment: kRelFlag | r
constexpr uint32_t kErrBarrier = 8u;         // barrier timeout (a peer never arrived)

int grid_n(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return static_cast<int>(b < 1 ? 1 : (b > 8192 ? 8192 : b));
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------- barrier
struct BarrierArgs {
  unsigned long long* flag_peer[8];  // rank k's flag array (G slots)
  unsigned long long* my_flags;      // this rank's array (= flag_peer[rank])
  unsigned long long* gen;           // this rank's generation counter
  uint32_t* err;                     // this rank's sticky error word
  int rank, world;
};

__global__ void shard_barrier_kernel(BarrierArgs b) {
  __shared__ unsigned long long gen;
  __shared__ int timed_out;
  const int t = threadIdx.x;
  if (t == 0) {
    gen = *b.gen + 1;
    *b.gen = gen;
    timed_out = 0;
  }
  __syncthreads();
  const uint32_t code = b.err[0];
  const unsigned long long mine =
      (gen << 32) | (code ? ((min(code, 255u) << 24) | (b.err[1] & 0xFFFFFFu)) : 0ull);
  // after a timeout a peer is gone: publish, never wait again (no 20 s per barrier)
  const bool gone = code == kErrBarrier;
  if (t < b.world) {
    __threadfence_system();  // this rank's stores of the phase before reach every peer first
    st_release_sys(b.flag_peer[t] + b.rank, mine);
    const unsigned long long t0 = gtimer();
    while (!gone && (ld_acquire_sys(b.my_flags + t) >> 32) < gen) {
      __nanosleep(64);
      if (gtimer() - t0 > 20000000000ull) {
        timed_out = 1;
        break;
      }
    }
  }
  __syncthreads();
  if (t == 0) {
    if (timed_out) {
      atomicCAS(&b.err[0], 0u, kErrBarrier);
    } else if (b.err[0] == 0) {  // adopt the error of the lowest failing rank
      for (int k = 0; k < b.world; ++k) {
        const uint32_t v = static_cast<uint32_t>(ld_acquire_sys(b.my_flags + k));
        if (v) {
          b.err[1] = v & 0xFFFFFFu;
          atomicCAS(&b.err[0], 0u, v >> 24);
          break;
        }
      }
    }
  }
}

// ---------------------------------------------------------------- plan kernels
// Forward pairs of this rank: {h, t, nh, nt} and r of its shard positions.
__global__ void shard_pairs_kernel(const int32_t* __restrict__ order_g, const int4* __restrict__ quad,
                                   const int32_t* __restrict__ R, int64_t Mg, int4* __restrict__ pair_ht,
                                   int32_t* __restrict__ pair_r) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < Mg;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t id = order_g[j];
    pair_ht[j] = quad[id];
    pair_r[j] = R[id];
  }
}

struct Geo {  // global batch geometry of the epoch
  int64_t M, B;  // train triples, global batch size
  int world, glog, rank;
};

// Position k of the epoch order -> batch b, index i, batch size Bb, the shard
// stride S_b of that batch and the rank / local row that computes pair i.
__device__ __forceinline__ void locate(const Geo& g, int64_t k, int64_t& b, int64_t& i, int64_t& Bb, int& owner,
                                       int64_t& lp, int64_t& Sk) {
  b = k / g.B;
  i = k - b * g.B;
  Bb = min(g.B, g.M - b * g.B);
  const int64_t S = (Bb + g.world - 1) / g.world;  // full batches: B / G exactly (B % G == 0)
  owner = static_cast<int>(i / S);
  lp = i - owner * S;
  Sk = min(S, Bb - owner * S);
}

__device__ __forceinline__ bool owns(int64_t id, const Geo& g) { return (id & ((1 << g.glog) - 1)) == g.rank; }

// Owned incidence entries of one row {h:+1, t:-1, r:+1}; the self-loop pair cancels (coo_to_csr).
__device__ __forceinline__ int owned_count(int32_t h, int32_t t, int32_t r, const Geo& g) {
  int c = owns(r, g) ? 1 : 0;
  if (h != t) c += (owns(h, g) ? 1 : 0) + (owns(t, g) ? 1 : 0);
  return c;
}

__global__ void shard_count_kernel(const int32_t* __restrict__ order, const int4* __restrict__ quad,
                                   const int32_t* __restrict__ R, Geo g, uint32_t* __restrict__ cnt) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < g.M;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t b, i, Bb, lp, Sk;
    int own;
    locate(g, k, b, i, Bb, own, lp, Sk);
    const int4 q = __ldg(quad + __ldg(order + k));
    const int32_t r = __ldg(R + __ldg(order + k));
    cnt[2 * b * g.B + i] = owned_count(q.x, q.y, r, g);
    cnt[2 * b * g.B + Bb + i] = owned_count(q.z, q.w, r, g);
  }
}

// Relation columns first inside a batch (long segments start early), then
// entities; both by local index.
__device__ __forceinline__ uint32_t shard_col_key(int64_t id, bool rel, int64_t nro, const Geo& g) {
  return static_cast<uint32_t>(rel ? (id >> g.glog) : nro + (id >> g.glog));
}

__global__ void shard_emit_kernel(const int32_t* __restrict__ order, const int4* __restrict__ quad,
                                  const int32_t* __restrict__ R, Geo g, int64_t nro, int cb,
                                  const uint32_t* __restrict__ off, uint32_t* __restrict__ key,
                                  uint32_t* __restrict__ val) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < g.M;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t b, i, Bb, lp, Sk;
    int own;
    locate(g, k, b, i, Bb, own, lp, Sk);
    const int4 q = __ldg(quad + __ldg(order + k));
    const int32_t r = __ldg(R + __ldg(order + k));
    const uint32_t bkey = static_cast<uint32_t>(b) << cb;
    const uint32_t who = static_cast<uint32_t>(own) << 28;
    for (int pass = 0; pass < 2; ++pass) {
      const int32_t h = pass ? q.z : q.x, t = pass ? q.w : q.y;
      const uint32_t lrow = static_cast<uint32_t>(pass ? Sk + lp : lp);  // row in the owner's residual buffer
      uint32_t o = off[2 * b * g.B + (pass ? Bb : 0) + i];
      if (h != t) {
        if (owns(h, g)) {
          key[o] = bkey | shard_col_key(h, false, nro, g);
          val[o++] = who | lrow;
        }
        if (owns(t, g)) {
          key[o] = bkey | shard_col_key(t, false, nro, g);
          val[o++] = 0x80000000u | who | lrow;
        }
      }
      if (owns(r, g)) {
        key[o] = bkey | shard_col_key(r, true, nro, g);
        val[o] = who | lrow;
      }
    }
  }
}

__global__ void shard_seg_flag_kernel(const uint32_t* __restrict__ key, int64_t E, uint32_t* __restrict__ flag) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < E;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    flag[e] = (e == 0 || key[e - 1] != key[e]) ? 1u : 0u;
}

__global__ void shard_seg_fill_kernel(const uint32_t* __restrict__ key, const uint32_t* __restrict__ flag,
                                      const uint32_t* __restrict__ segid, int64_t E, int cb, int64_t nro, Geo g,
                                      int64_t nb, const uint32_t* __restrict__ nseg, uint32_t* __restrict__ seg_start,
                                      uint32_t* __restrict__ seg_col, uint32_t* __restrict__ seg_base) {
  const uint32_t cmask = (1u << cb) - 1u;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < E;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t k = key[e];
    if (flag[e]) {
      const uint32_t sidx = segid[e];
      seg_start[sidx] = static_cast<uint32_t>(e);
      const int64_t cp = k & cmask;
      // relation: global id (local index * G + rank); entity: local row
      seg_col[sidx] = cp < nro ? (kRelFlag | static_cast<uint32_t>((cp << g.glog) | g.rank))
                               : static_cast<uint32_t>(cp - nro);
      const uint32_t b = k >> cb;
      if (e == 0 || (key[e - 1] >> cb) != b)
        for (uint32_t bb = e == 0 ? 0u : (key[e - 1] >> cb) + 1; bb <= b; ++bb) seg_base[bb] = sidx;
    }
    if (e + 1 == E) {
      seg_start[*nseg] = static_cast<uint32_t>(E);
      for (int64_t bb = (k >> cb) + 1; bb <= nb; ++bb) seg_base[bb] = *nseg;
    }
  }
}

__global__ void empty_plan_kernel(uint32_t* __restrict__ seg_base, int64_t nb, uint32_t* __restrict__ seg_start) {
  for (int64_t b = threadIdx.x; b <= nb; b += blockDim.x) seg_base[b] = 0;
  if (threadIdx.x == 0) seg_start[0] = 0;
}

// ---------------------------------------------------------------- backward
struct SegArgs {
  float* ent;                   // this rank's entity shard (updated in place)
  float* rel_peer[8];           // every rank's relation replica (the owner writes all)
  const float* res_peer[8];     // residual rows of every rank
  const float* scal_peer[8];    // row scales of every rank
  const uint32_t* ent_val;      // sorted entries: sign << 31 | rank << 28 | local row
  const uint32_t* seg_start;
  const uint32_t* seg_col;
  const uint32_t* seg_base;
  int batch, d, world;
  const float* lr;
  const uint32_t* err;
};

template <int KIND>
__device__ __forceinline__ float dir1s(float r, float sc) {  // models.cpp:37-60, norms.hpp:119-126
  if (KIND == kTransE_L2 || KIND == kTorusE_L2) return __fmul_rn(r, sc);
  return r > 0.f ? sc : (r < 0.f ? -sc : 0.f);
}

// One warp per owned column segment: acc = sum of a * D_row in entry order
// (the reference's ascending-row order), then p - lr * acc. Relation rows are
// written to every replica. Up to 4 residual rows (peer loads) in flight.
template <int KIND, int CH>
__global__ void __launch_bounds__(256) shard_segment_kernel(const SegArgs a) {
  if (a.err[0] != 0) return;
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (blockDim.x >> 5);
  const uint32_t s0 = a.seg_base[a.batch], s1 = a.seg_base[a.batch + 1];
  const int dv = a.d >> 2;
  const float lr = *a.lr;
  for (uint32_t s = s0 + gw; s < s1; s += nw) {
    const uint32_t col = a.seg_col[s];
    const uint32_t e0 = a.seg_start[s], e1 = a.seg_start[s + 1];
    const bool rel = (col & kRelFlag) != 0;
    const size_t row = col & ~kRelFlag;
    float4* P = reinterpret_cast<float4*>(rel ? a.rel_peer[0] : a.ent) + row * dv;  // replicas are identical
    for (int cb = 0; cb < dv; cb += 32 * CH) {
      int c[CH];
      bool has[CH];
      float4 acc[CH], p[CH];
#pragma unroll
      for (int h = 0; h < CH; ++h) {
        c[h] = cb + 32 * h + lane;
        has[h] = c[h] < dv;
        acc[h] = make_float4(0.f, 0.f, 0.f, 0.f);
        p[h] = has[h] ? P[c[h]] : acc[h];
      }
      for (uint32_t eb = e0; eb < e1; eb += 32) {
        const int cnt = min(32u, e1 - eb);
        uint32_t myv = 0;
        float mysc = 0.f;
        if (lane < cnt) {
          myv = a.ent_val[eb + lane];
          mysc = a.scal_peer[(myv >> 28) & 7u][myv & 0x0FFFFFFFu];
        }
        unsigned live = __ballot_sync(kFull, lane < cnt && mysc != 0.f);
        while (live) {
          constexpr int KB = 4;
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
          float4 rv[KB][CH];
#pragma unroll
          for (int q = 0; q < KB; ++q) {
            vq[q] = __shfl_sync(kFull, myv, k[q]);
            scq[q] = __shfl_sync(kFull, mysc, k[q]);
            const float4* R4 = reinterpret_cast<const float4*>(a.res_peer[(vq[q] >> 28) & 7u]) +
                               static_cast<size_t>(vq[q] & 0x0FFFFFFFu) * dv;
#pragma unroll
            for (int h = 0; h < CH; ++h)
              if (q < n && has[h]) rv[q][h] = __ldg(R4 + c[h]);
          }
#pragma unroll
          for (int q = 0; q < KB; ++q)
            if (q < n) {
              const bool neg = (vq[q] >> 31) != 0;
#pragma unroll
              for (int h = 0; h < CH; ++h)
                if (has[h]) {
                  float* A = &acc[h].x;
                  const float* V = &rv[q][h].x;
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    const float x = dir1s<KIND>(V[e], scq[q]);
                    A[e] = __fadd_rn(A[e], neg ? -x : x);  // sparse.hpp:284-296 association
                  }
                }
            }
        }
      }
#pragma unroll
      for (int h = 0; h < CH; ++h) {
        if (!has[h]) continue;
        float4 np;  // embedding.cpp:177-178: p - lr * g, no FMA
        np.x = __fsub_rn(p[h].x, __fmul_rn(lr, acc[h].x));
        np.y = __fsub_rn(p[h].y, __fmul_rn(lr, acc[h].y));
        np.z = __fsub_rn(p[h].z, __fmul_rn(lr, acc[h].z));
        np.w = __fsub_rn(p[h].w, __fmul_rn(lr, acc[h].w));
        if (rel) {
          for (int k = 0; k < a.world; ++k) reinterpret_cast<float4*>(a.rel_peer[k])[row * dv + c[h]] = np;
        } else {
          P[c[h]] = np;
        }
      }
    }
  }
  __threadfence_system();  // peer stores visible before this rank's next barrier
}

// Global batch loss = sum over ranks (rank order) of the shards' loss / Bb.
__global__ void shard_loss_kernel(const float* const* __restrict__ loss_peer_dev, int world, int64_t nb,
                                  float* __restrict__ out) {
  for (int64_t b = threadIdx.x; b < nb; b += blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < world; ++k) s = __fadd_rn(s, loss_peer_dev[k][b]);
    out[b] = s;
  }
}

// Entity shard <-> full table (store upload / download in shard mode).
__global__ void scatter_owned_kernel(const float* __restrict__ full, int64_t n_own, int64_t d, int glog, int rank,
                                     float* __restrict__ shard) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n_own * d;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t lr = i / d, j = i - lr * d;
    shard[i] = full[((lr << glog) | rank) * d + j];
  }
}
__global__ void gather_full_kernel(ShardPtrs p, int64_t N, int64_t d, int glog, float* __restrict__ full) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N * d;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e = i / d, j = i - e * d;
    full[i] = p.ent[e & ((1 << glog) - 1)][(e >> glog) * d + j];
  }
}

int64_t owned_rows(int64_t n, int world, int rank) { return n > rank ? (n - rank + world - 1) / world : 0; }

}  // namespace

// ---------------------------------------------------------------- state

void ShardPlanBufs::reserve(int64_t pairs, int64_t rows2, int64_t entries, int64_t batches) {
  if (pairs > cap_pairs) {
    if (pair_ht) cudaFree(pair_ht);
    if (pair_r) cudaFree(pair_r);
    SKG_CUDA(cudaMalloc(&pair_ht, sizeof(int4) * (pairs + 1)));
    SKG_CUDA(cudaMalloc(&pair_r, sizeof(int32_t) * (pairs + 1)));
    cap_pairs = pairs;
  }
  if (rows2 > cap_rows) {
    if (cnt) cudaFree(cnt);
    if (off) cudaFree(off);
    SKG_CUDA(cudaMalloc(&cnt, sizeof(uint32_t) * (rows2 + 1)));
    SKG_CUDA(cudaMalloc(&off, sizeof(uint32_t) * (rows2 + 1)));
    cap_rows = rows2;
    scan.reserve(std::max(rows2, cap_entries));
  }
  if (entries > cap_entries) {
    for (uint32_t** b : {&key, &val, &key_alt, &val_alt, &seg_start, &seg_col}) {
      if (*b) cudaFree(*b);
      SKG_CUDA(cudaMalloc(b, sizeof(uint32_t) * (entries + 1)));
    }
    cap_entries = entries;
    sort.reserve(entries);
    scan.reserve(std::max(rows2, cap_entries));
  }
  if (batches > cap_batches) {
    if (seg_base) cudaFree(seg_base);
    SKG_CUDA(cudaMalloc(&seg_base, sizeof(uint32_t) * (batches + 1)));
    cap_batches = batches;
  }
  if (!nseg) SKG_CUDA(cudaMalloc(&nseg, sizeof(uint32_t)));
}

void ShardPlanBufs::release() {
  for (void* b : {static_cast<void*>(pair_ht), static_cast<void*>(pair_r), static_cast<void*>(cnt),
                  static_cast<void*>(off), static_cast<void*>(key), static_cast<void*>(val),
                  static_cast<void*>(key_alt), static_cast<void*>(val_alt), static_cast<void*>(seg_start),
                  static_cast<void*>(seg_col), static_cast<void*>(seg_base), static_cast<void*>(nseg)})
    if (b) cudaFree(b);
  pair_ht = nullptr;
  pair_r = nullptr;
  cnt = off = key = val = key_alt = val_alt = seg_start = seg_col = seg_base = nseg = nullptr;
  cap_pairs = cap_rows = cap_entries = cap_batches = 0;
  sort.release();
  scan.release();
}

ShardState::~ShardState() {
  for (int k = 0; k < world; ++k)
    if (opened[k]) cudaIpcCloseMemHandle(opened[k]);
  if (arena) cudaFree(arena);
  if (ptr_dev) cudaFree(ptr_dev);
}

// Arena layout (byte offsets, 256-aligned): entity shard | relation replica |
// residual rows | row scales | shard losses | barrier flags + generation.
void shard_alloc(skg_ctx* ctx, int rank, int world, int64_t batch_size) {
  if (ctx->shard) throw ConfigError("sharded tables already initialised on this context");
  if (world != 1 && world != 2 && world != 4 && world != 8)
    throw ConfigError("sharded data parallel: world must be 1, 2, 4 or 8");
  if (rank < 0 || rank >= world) throw ConfigError("sharded data parallel: bad rank");
  if (!ctx->has_store) throw ConfigError("no parameter store uploaded");
  if (ctx->cfg.model != SKG_TRANSE && ctx->cfg.model != SKG_TORUSE)
    throw ConfigError("sharded data parallel covers the hrt models (transe, toruse)");
  if (ctx->de % 4 != 0) throw ConfigError("sharded tables need an embedding dimension divisible by 4");
  if (batch_size < world || batch_size % world != 0)
    throw ConfigError("data parallel: global batch_size must be a multiple of the world size");
  auto* st = new ShardState();
  st->rank = rank;
  st->world = world;
  st->glog = world == 1 ? 0 : world == 2 ? 1 : world == 4 ? 2 : 3;
  st->B = batch_size;
  st->d = ctx->de;
  st->NEo = owned_rows(ctx->N, world, rank);
  st->NRo = owned_rows(ctx->R, world, rank);
  st->S = batch_size / world;
  st->nb_cap = (std::max<int64_t>(ctx->M, 1) + batch_size - 1) / batch_size + 1;
  auto al = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
  size_t o = 0;
  // every rank uses the same layout (peers' buffers are addressed with this
  // rank's offsets): the entity region holds ceil(N / G) rows on all ranks
  const int64_t ne_cap = (ctx->N + world - 1) / world;
  st->off_ent = o;
  o += al(sizeof(float) * ne_cap * st->d + 16);
  st->off_rel = o;
  o += al(sizeof(float) * ctx->R * st->d);
  st->off_res = o;
  o += al(sizeof(float) * 2 * st->S * st->d);
  st->off_scal = o;
  o += al(sizeof(float) * 2 * st->S);
  st->off_loss = o;
  o += al(sizeof(float) * st->nb_cap);
  st->off_flags = o;
  o += al(sizeof(unsigned long long) * (world + 1));
  st->arena_bytes = o;
  SKG_CUDA(cudaMalloc(&st->arena, o));
  SKG_CUDA(cudaMemset(st->arena, 0, o));
  SKG_CUDA(cudaMalloc(&st->ptr_dev, sizeof(float*) * 8));
  ctx->shard = st;
  // the owned entity rows and the relation replica from the uploaded store
  shard_scatter_store(ctx);
}

void shard_scatter_store(skg_ctx* ctx) {
  ShardState* st = ctx->shard;
  char* A = static_cast<char*>(st->arena);
  if (st->NEo > 0)
    scatter_owned_kernel<<<grid_n(st->NEo * st->d), 256, 0, ctx->stream>>>(
        ctx->tables.p, st->NEo, st->d, st->glog, st->rank, reinterpret_cast<float*>(A + st->off_ent));
  SKG_CUDA(cudaMemcpyAsync(A + st->off_rel, ctx->tables.p + ctx->N * ctx->de, sizeof(float) * ctx->R * ctx->dr,
                           cudaMemcpyDeviceToDevice, ctx->stream));
  count_launch();
  SKG_LAUNCH_CHECK();
  SKG_CUDA(cudaStreamSynchronize(ctx->stream));
}

// Full entity / relation tables into ctx->tables (store download in shard mode).
void shard_gather_store(skg_ctx* ctx) {
  ShardState* st = ctx->shard;
  gather_full_kernel<<<grid_n(ctx->N * st->d), 256, 0, ctx->stream>>>(st->peers, ctx->N, st->d, st->glog,
                                                                      ctx->tables.p);
  SKG_CUDA(cudaMemcpyAsync(ctx->tables.p + ctx->N * ctx->de, st->peers.rel[st->rank],
                           sizeof(float) * ctx->R * ctx->dr, cudaMemcpyDeviceToDevice, ctx->stream));
  count_launch();
  SKG_LAUNCH_CHECK();
  SKG_CUDA(cudaStreamSynchronize(ctx->stream));
}

// Resolves every rank's arena base into the typed peer pointers.
void shard_link(skg_ctx* ctx, void* const* bases) {
  ShardState* st = ctx->shard;
  for (int k = 0; k < st->world; ++k) {
    char* A = static_cast<char*>(bases[k]);
    st->peers.ent[k] = reinterpret_cast<float*>(A + st->off_ent);
    st->peers.rel[k] = reinterpret_cast<float*>(A + st->off_rel);
    st->peers.res[k] = reinterpret_cast<float*>(A + st->off_res);
    st->peers.scal[k] = reinterpret_cast<float*>(A + st->off_scal);
    st->peers.loss[k] = reinterpret_cast<float*>(A + st->off_loss);
    st->peers.flags[k] = reinterpret_cast<unsigned long long*>(A + st->off_flags);
  }
  SKG_CUDA(cudaMemcpy(st->ptr_dev, st->peers.loss, sizeof(float*) * 8, cudaMemcpyHostToDevice));
  st->linked = true;
  drop_graphs(ctx);
}

// The owned-entry count of an epoch depends on the data only (every epoch
// permutes the same rows), so the plan size is fixed per data version; it is
// computed outside graph capture and kept on the host.
int64_t shard_entry_count(skg_ctx* ctx) {
  ShardState* st = ctx->shard;
  if (st->count_version == ctx->data_version) return st->E;
  Geo g{ctx->M, st->B, st->world, st->glog, st->rank};
  ShardPlanBufs& p = st->plan[0];
  p.reserve(0, 2 * ctx->M, 0, 1);
  DevBuf<int32_t> iota;
  iota.ensure(ctx->M + 1);
  device_iota(iota.p, ctx->M, ctx->stream);
  shard_count_kernel<<<grid_n(ctx->M), 256, 0, ctx->stream>>>(iota.p, ctx->quad.p, ctx->Rl.p, g, p.cnt);
  count_launch();
  SKG_LAUNCH_CHECK();
  DevBuf<uint32_t> tot;
  tot.ensure(1);
  ScanPlan sc;
  sc.reserve(2 * ctx->M);
  exclusive_scan_u32(p.cnt, p.cnt, 2 * ctx->M, tot.p, sc, ctx->stream);
  uint32_t E = 0;
  SKG_CUDA(cudaMemcpyAsync(&E, tot.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
  SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  st->E = E;
  st->count_version = ctx->data_version;
  return E;
}

// This rank's forward pairs and its owned-entry plan of one epoch (slot).
void shard_build_plan(skg_ctx* ctx, const int32_t* order, const int32_t* order_g, int64_t Mg, int slot,
                      cudaStream_t s) {
  ShardState* st = ctx->shard;
  ShardPlanBufs& p = st->plan[slot];
  Geo g{ctx->M, st->B, st->world, st->glog, st->rank};
  const int64_t nb = (ctx->M + st->B - 1) / st->B;
  const int64_t E = st->E;
  p.reserve(Mg, 2 * ctx->M, E, nb);
  p.nb = nb;
  p.E = E;
  if (Mg > 0) {
    shard_pairs_kernel<<<grid_n(Mg), 256, 0, s>>>(order_g, ctx->quad.p, ctx->Rl.p, Mg, p.pair_ht, p.pair_r);
    count_launch();
    SKG_LAUNCH_CHECK();
  }
  if (E == 0) {
    empty_plan_kernel<<<1, 256, 0, s>>>(p.seg_base, nb, p.seg_start);
    count_launch();
    SKG_LAUNCH_CHECK();
    p.sorted_val = p.val;
    return;
  }
  const int cb = bits_for(static_cast<uint64_t>(st->NRo + st->NEo));
  const int kb = bits_for(static_cast<uint64_t>(nb - 1));
  if (kb + cb > 31) throw CudaError("shard plan: batches x owned columns exceed the 31-bit key space");
  shard_count_kernel<<<grid_n(ctx->M), 256, 0, s>>>(order, ctx->quad.p, ctx->Rl.p, g, p.cnt);
  exclusive_scan_u32(p.cnt, p.off, 2 * ctx->M, nullptr, p.scan, s);
  shard_emit_kernel<<<grid_n(ctx->M), 256, 0, s>>>(order, ctx->quad.p, ctx->Rl.p, g, st->NRo, cb, p.off, p.key,
                                                   p.val);
  count_launch(2);
  SKG_LAUNCH_CHECK();
  const bool alt = radix_sort_pairs(p.key, p.val, p.key_alt, p.val_alt, E, kb + cb, p.sort, s);
  const uint32_t* k = alt ? p.key_alt : p.key;
  p.sorted_val = alt ? p.val_alt : p.val;
  uint32_t* flag = alt ? p.key : p.key_alt;
  uint32_t* segid = alt ? p.val : p.val_alt;
  shard_seg_flag_kernel<<<grid_n(E), 256, 0, s>>>(k, E, flag);
  exclusive_scan_u32(flag, segid, E, p.nseg, p.scan, s);
  shard_seg_fill_kernel<<<grid_n(E), 256, 0, s>>>(k, flag, segid, E, cb, st->NRo, g, nb, p.nseg, p.seg_start,
                                                  p.seg_col, p.seg_base);
  count_launch(2);
  SKG_LAUNCH_CHECK();
}

void shard_barrier(skg_ctx* ctx, cudaStream_t s) {
  ShardState* st = ctx->shard;
  BarrierArgs b{};
  for (int k = 0; k < st->world; ++k) b.flag_peer[k] = st->peers.flags[k];
  b.my_flags = st->peers.flags[st->rank];
  b.gen = st->peers.flags[st->rank] + st->world;
  b.err = ctx->err_words.p;
  b.rank = st->rank;
  b.world = st->world;
  shard_barrier_kernel<<<1, 32, 0, s>>>(b);
  count_launch();
  SKG_LAUNCH_CHECK();
}

void shard_backward(skg_ctx* ctx, int kind, int slot, int64_t batch, cudaStream_t s) {
  ShardState* st = ctx->shard;
  const ShardPlanBufs& p = st->plan[slot];
  SegArgs a{};
  a.ent = st->peers.ent[st->rank];
  for (int k = 0; k < st->world; ++k) {
    a.res_peer[k] = st->peers.res[k];
    a.scal_peer[k] = st->peers.scal[k];
  }
  // rel_peer[0] is this rank's replica (the row read); the owner writes all G
  for (int k = 0; k < st->world; ++k) a.rel_peer[k] = st->peers.rel[(st->rank + k) % st->world];
  a.ent_val = p.sorted_val;
  a.seg_start = p.seg_start;
  a.seg_col = p.seg_col;
  a.seg_base = p.seg_base;
  a.batch = static_cast<int>(batch);
  a.d = static_cast<int>(st->d);
  a.world = st->world;
  a.lr = ctx->lr_dev.p;
  a.err = ctx->err_words.p;
  const int grid = ctx->num_sms * 8;
  const bool wide = st->d > 128;
  switch (kind) {
#define SKG_SHARD_SEG(K)                                                                     \
  case K:                                                                                    \
    if (wide) shard_segment_kernel<K, 2><<<grid, 256, 0, s>>>(a);                            \
    else shard_segment_kernel<K, 1><<<grid, 256, 0, s>>>(a);                                 \
    break;
    SKG_SHARD_SEG(kTransE_L2)
    SKG_SHARD_SEG(kTransE_L1)
    SKG_SHARD_SEG(kTorusE_L2)
    SKG_SHARD_SEG(kTorusE_L1)
#undef SKG_SHARD_SEG
    default: throw ConfigError("sharded data parallel covers the hrt models (transe, toruse)");
  }
  count_launch();
  SKG_LAUNCH_CHECK();
}

void shard_finish_losses(skg_ctx* ctx, int64_t nb, cudaStream_t s) {
  ShardState* st = ctx->shard;
  shard_loss_kernel<<<1, 256, 0, s>>>(st->ptr_dev, st->world, nb, ctx->batch_loss.p);
  count_launch();
  SKG_LAUNCH_CHECK();
}

void shard_fill_fwd(skg_ctx* ctx, FwdArgs& fa) {
  ShardState* st = ctx->shard;
  for (int k = 0; k < 8; ++k) fa.ent_peer[k] = k < st->world ? st->peers.ent[k] : st->peers.ent[0];
  fa.glog = st->glog;
  fa.rel_rows = st->peers.rel[st->rank];
  fa.X = nullptr;
  fa.res = st->peers.res[st->rank];
  fa.scal = st->peers.scal[st->rank];
  fa.batch_loss = st->peers.loss[st->rank];
}

void shard_destroy(skg_ctx* ctx) {
  if (!ctx->shard) return;
  drop_graphs(ctx);
  cudaDeviceSynchronize();
  delete ctx->shard;
  ctx->shard = nullptr;
}

}  // namespace skg

namespace skg {
// Identity of the sharded buffers baked into a captured epoch graph.
uint64_t shard_tag(const skg_ctx* ctx) {
  const ShardState* st = ctx->shard;
  if (!st) return 0;
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
  for (const auto& p : st->plan)
    for (const void* q : {static_cast<const void*>(p.pair_ht), static_cast<const void*>(p.pair_r),
                          static_cast<const void*>(p.cnt), static_cast<const void*>(p.off),
                          static_cast<const void*>(p.key), static_cast<const void*>(p.val),
                          static_cast<const void*>(p.key_alt), static_cast<const void*>(p.val_alt),
                          static_cast<const void*>(p.seg_start), static_cast<const void*>(p.seg_col),
                          static_cast<const void*>(p.seg_base), static_cast<const void*>(p.nseg)})
      mix(reinterpret_cast<uintptr_t>(q));
  mix(static_cast<uint64_t>(st->E));
  mix(reinterpret_cast<uintptr_t>(st->arena));
  mix(st->linked);
  for (int k = 0; k < st->world; ++k) mix(reinterpret_cast<uintptr_t>(st->peers.ent[k]));
  return h;
}
int shard_rank(const skg_ctx* ctx) { return ctx->shard ? ctx->shard->rank : 0; }
int shard_world(const skg_ctx* ctx) { return ctx->shard ? ctx->shard->world : 1; }
}  // namespace skg
