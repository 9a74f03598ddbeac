// TransR training step on tcgen05, warp-specialized (sm_100a), d_e = d_r = 128.
//
// Per tile of 64 (pos, neg) pairs = 128 rows of one relation r
// (models.cpp:110-156, models.hpp:82-96):
//   U  = h - t                        gathered by the producer warps
//   V  = U M_r^T          (GEMM1)     V_row + r -> reference-order score, hinge
//   DZ = dir(V + r) * up              epilogue warps
//   dM += DZ^T U          (GEMM3)     accumulated in TMEM over the relation run
//   dU  = DZ M_r          (GEMM2)     -> res_u rows for the entity segments
// All three products are 3xTF32 (hi*hi + hi*lo + lo*hi, fp32-class). The
// tensor core truncates a raw fp32 operand to tf32, so raw U / DZ serve as the
// "hi" A operands and only lo = x - trunc(x) is materialised; GEMM1 / GEMM2
// read both from TMEM (tcgen05.mma [a_tmem]). M_r arrives pre-split (hi =
// rna, lo = rest) in 16-wide K chunks through a 3-slot bulk-copy ring; GEMM3
// contracts over rows, so DZ^T / U^T are staged 8 rows at a time from the
// shared-memory copies of U and DZ.
//
// Roles (320 threads):
//   warps 0-3  epilogue   thread = row = TMEM lane: score, hinge, DZ, sum(dz),
//                         dM flush per relation run, dU drain to HBM
//   warps 4-7  producer   row-id chase, U gather, U lo -> TMEM, G3 staging
//   warp  8    MMA issue  (whole warp, elect.sync inside the asm)
//   warp  9    ring loader (bulk copies of M_r chunks)
//   warp 10    row-id chase (tile -> incidence rows -> head / tail), two tiles ahead
// TMEM columns: see kColHi .. kColDM below.
//
// The CTA-range / relation-run partition (slot = CTA + run ordinal) is the one
// transr_tc_apply_kernel (transr_tc.cu) reduces in tile order.
#include "common.cuh"
#include "ht.cuh"
#include "primitives.cuh"
#include "refmath.cuh"
#include "tc.cuh"

namespace skg {

namespace {

constexpr int kD = 128;
constexpr int kRows = 128;
constexpr int kPairs = 64;
#ifndef SKG_TR_GATHER_WARPS
#define SKG_TR_GATHER_WARPS 4
#endif
constexpr int kGatherWarps = SKG_TR_GATHER_WARPS;  // one warp's cp.async stream cannot fill an SM's L2 bandwidth
constexpr int kMmaWarp = 8, kRowWarp = 10, kGatherWarp = 11;  // warp 9: ring loader; gather warps 11 ..
constexpr int kThreads = (kGatherWarp + kGatherWarps) * 32;

// sU / sDZ: row tiles (m = row, feature) in four 32-feature column blocks of
// 128 rows x 128 B, 32-byte chunks XOR-swizzled by (row & 3): the
// SWIZZLE_128B_BASE32B layout, so GEMM3 reads both tiles in place as MN-major
// operands (K = rows, MN = features; LBO = the 16 KB block stride, SBO = 512 B
// per 4 rows — tools/umma_mn_probe.cu). 16-byte unit (r, c4) =
// block * 1024 + r * 8 + (((c4 & 7) >> 1) ^ (r & 3)) * 2 + (c4 & 1).
__device__ __forceinline__ int swz32(int r, int c4) { return ((((c4 & 7) >> 1) ^ (r & 3)) << 1) | (c4 & 1); }
__device__ __forceinline__ int tile_unit(int r, int c4) { return (c4 >> 3) * 1024 + r * 8 + swz32(r, c4); }
constexpr uint32_t kTileLBO = 1024 * 16, kSBO32 = 4 * 128;


// Ring chunk of M_r: 128 (n) x 16 (k), hi then lo; unit (n, k4) = (n & 7) + (n >> 3) * 32 + k4 * 8.
constexpr int kChunkK = 16;
constexpr int kChunkFloats = kD * kChunkK;
constexpr uint32_t kChunkBytes = 2 * kChunkFloats * sizeof(float);
constexpr uint32_t kChLBO = 8 * 16, kChSBO = 32 * 16;
constexpr int kChunksPerGemm = kD / kChunkK;
constexpr int64_t kMrFloatsPerRel = 2LL * kChunksPerGemm * 2 * kChunkFloats;
constexpr int kRing = 3;
#ifndef SKG_APPLY_Y
#define SKG_APPLY_Y 32  // relation-parallel blocks x 32 slices of the 16 K-element proj block
#endif

// GEMM3 (dM += DZ^T U, K = rows) in slots of 8 rows: the hi terms are the raw
// sDZ / sU rows read in place (the tensor core truncates fp32 to tf32); only
// lo = x - trunc(x) of DZ and U is staged, row-major in the same swizzle
// (8 rows x 4 blocks of 128 B: LBO = 1 KB, SBO = 512 B), no transposition.
constexpr int kG3Rows = 8;
constexpr int kG3ArrFloats = kG3Rows * kD;
constexpr uint32_t kG3LBO = kG3Rows * 128;
#ifndef SKG_TR_G3_SLOTS
#define SKG_TR_G3_SLOTS 4
#endif
constexpr int kG3Slots = SKG_TR_G3_SLOTS;
constexpr int kG3PerTile = kRows / kG3Rows;
__device__ __forceinline__ int g3_unit(int r, int c4) { return (c4 >> 3) * (kG3Rows * 8) + r * 8 + swz32(r, c4); }

// TMEM columns: [0,128) U hi -> DZ hi and [128,256) U lo -> DZ lo (A operands
// of GEMM1 / GEMM2 read straight from TMEM), [256,384) V, then dU (GEMM2
// writes dU over the consumed V; GEMM1 of the next tile waits for the drain),
// [384,512) dM.
constexpr uint32_t kColHi = 0, kColLo = 128, kColV = 256, kColDU = 256, kColDM = 384;

// Phase timestamps (clock64) for pipeline analysis, off unless enabled through
// skg_debug_transr_trace: [CTA][tile < 16][event < 16].
constexpr int kTrCtas = 160, kTrTiles = 16, kTrEvents = 16;
__device__ unsigned long long g_trace[kTrCtas * kTrTiles * kTrEvents];
__device__ int g_trace_on;
__device__ __forceinline__ void trace_ev(bool on, uint32_t it, int ev) {
  if (on && it < kTrTiles && blockIdx.x < kTrCtas && (threadIdx.x & 31) == 0)
    g_trace[(blockIdx.x * kTrTiles + it) * kTrEvents + ev] = clock64();
}

struct Smem {
  float U[kRows * kD];
  float DZ[kRows * kD];
  float ring[kRing][2 * kChunkFloats];
  float g3[kG3Slots][2][kG3ArrFloats];  // DZ lo, U lo (1 KB-aligned slots)
  int4 rows[2][kRows];                  // {head, tail, incidence row (-1: padding), 0}
  float rel[2][kD];
  int np[2];
  float rs[kRows];
  float sc[kRows];  // per-row gradient scale of the current tile (pass 2 of the producers)
  float colsum[4][kD];
  float tl[2];
  uint64_t g_full, v_full, dz_full, g2_done, du_empty, dm_full, dm_empty, sc_full;
  uint64_t u_q[4];  // U columns [32 q, 32 q + 32) in TMEM: GEMM1 starts on the first K quarter
  uint64_t rows_full[2], rows_empty[2];
  uint64_t g3_full[kG3Slots], g3_empty[kG3Slots];
  uint64_t stg[kRows / 8];  // row group s consumed by GEMM3: its sU / sDZ rows may be refilled
  uint64_t ring_full[kRing], ring_empty[kRing];
  uint32_t tmem_base;
  int last;
};

struct Args {
  FwdArgs f;
  const uint32_t* ent_val;
  const uint32_t* seg_start;
  const uint32_t* seg_col;
  const uint32_t* tile_seg;
  const uint32_t* tile_p0;
  const uint32_t* tile_total;  // [0] tiles, [1] relation segments
  const uint32_t* seg_tiles;
  float* dm_part;
  float* dr_part;
  const float* mr;  // per relation: [layout][chunk][hi, lo][128 x 16]
};

__device__ __forceinline__ void st_global_v8(float* p, const uint32_t* v) {  // one 32-byte store
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

// lo = x - trunc(x) of slot s3's 8 rows of DZ and U into ring slot (it * 16 + s3) % kG3Slots;
// thread t < 128: row t >> 4 of the slot, 16-byte units t & 15 and (t & 15) + 16.
#ifndef SKG_TR_STAGE_STEP
#define SKG_TR_STAGE_STEP 2
#endif
constexpr int kStageStep = SKG_TR_STAGE_STEP;  // 2: producers stage even slots, epilogue warps odd ones
__device__ __forceinline__ void stage_slot(Smem& S, uint32_t it, int s3, int t) {
  const uint32_t g3n = it * kG3PerTile + static_cast<uint32_t>(s3);
  const int slot = static_cast<int>(g3n % kG3Slots);
  if (g3n >= kG3Slots) tc::mbar_wait(&S.g3_empty[slot], ((g3n / kG3Slots) - 1) & 1);
  const int rq = t >> 4, cq = t & 15;
  const int row = s3 * kG3Rows + rq;
  float* Alo = S.g3[slot][0];
  float* Blo = S.g3[slot][1];
#pragma unroll
  for (int h2 = 0; h2 < 2; ++h2) {
    const int c4 = cq + 16 * h2;
    const float4 dz = *reinterpret_cast<const float4*>(S.DZ + 4 * tile_unit(row, c4));
    const float4 u = *reinterpret_cast<const float4*>(S.U + 4 * tile_unit(row, c4));
    const int o = 4 * g3_unit(rq, c4);
    *reinterpret_cast<float4*>(Alo + o) = make_float4(tc::tf32_trunc_lo(dz.x), tc::tf32_trunc_lo(dz.y),
                                                      tc::tf32_trunc_lo(dz.z), tc::tf32_trunc_lo(dz.w));
    *reinterpret_cast<float4*>(Blo + o) = make_float4(tc::tf32_trunc_lo(u.x), tc::tf32_trunc_lo(u.y),
                                                      tc::tf32_trunc_lo(u.z), tc::tf32_trunc_lo(u.w));
  }
  tc::fence_async_shared();
  tc::mbar_arrive(&S.g3_full[slot]);
}

__device__ __forceinline__ float4 f4sel(int c, float4 a, float4 b) {  // c ? a : b
  return make_float4(c ? a.x : b.x, c ? a.y : b.y, c ? a.z : b.z, c ? a.w : b.w);
}

// U = h - t in place for row p, columns [c0, c1), hi / lo -> TMEM lane p
// (taddr carries the warp's lane quadrant). Rows p and p + 4 share a swizzled
// 32-byte chunk: rows with bit 2 set visit the two 16-byte units of each chunk
// in swapped order, so the eight rows of a quarter-warp phase touch eight
// distinct units.
__device__ __forceinline__ void compute_u(Smem& S, uint32_t taddr, int p, bool ok_row, int c0, int c1, int de) {
  const int flip = (p >> 2) & 1;
#pragma unroll 1
  for (int c = c0; c < c1; c += 16) {
    const bool ok = ok_row && c < de;  // d_e is a multiple of 16: whole chunks are real or padding
    float hi[16], lo[16];
    float4 uv[4];
#pragma unroll
    for (int q = 0; q < 16; q += 4) {
      const int j = (q >> 2) ^ flip;
      float4* up = reinterpret_cast<float4*>(S.U + 4 * tile_unit(p, (c >> 2) + j));
      const float4 xh = *up;
      const float4 xt = *reinterpret_cast<const float4*>(S.DZ + 4 * tile_unit(p, (c >> 2) + j));
      const float4 u = ok ? make_float4(__fsub_rn(xh.x, xt.x), __fsub_rn(xh.y, xt.y), __fsub_rn(xh.z, xt.z),
                                        __fsub_rn(xh.w, xt.w))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
      *up = u;
      uv[q >> 2] = u;
    }
#pragma unroll
    for (int q = 0; q < 16; q += 4) {
      const float4 u = f4sel(flip, uv[(q >> 2) ^ 1], uv[q >> 2]);
      hi[q] = u.x, hi[q + 1] = u.y, hi[q + 2] = u.z, hi[q + 3] = u.w;
      lo[q] = tc::tf32_trunc_lo(u.x);
      lo[q + 1] = tc::tf32_trunc_lo(u.y);
      lo[q + 2] = tc::tf32_trunc_lo(u.z);
      lo[q + 3] = tc::tf32_trunc_lo(u.w);
    }
    tc::tmem_st16(taddr + kColHi + c, hi);
    tc::tmem_st16(taddr + kColLo + c, lo);
  }
}

// Pass 2 of the epilogue for row m, columns [c0, c1): DZ = dir(V + r) * sc
// -> sDZ (raw = tf32 hi) and TMEM hi / lo, column sums of the warp's 32 rows
// -> colsum[w][c]. Unit pairs in swapped order on rows with bit 2 set (see
// compute_u).
#ifndef SKG_TR_DZSPLIT
#define SKG_TR_DZSPLIT 64
#endif
constexpr int kDzSplit = SKG_TR_DZSPLIT;  // epilogue warps: columns [0, kDzSplit); producers: the rest
template <bool L2>
__device__ __forceinline__ void dz_pass(Smem& S, uint32_t taddr, int m, int w, float sc, const float* relr, int c0,
                                        int c1) {
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int c = c0; c < c1; c += 32) {
    uint32_t r0[16], r1[16];
    tc::tmem_ld16_nowait(taddr + kColV + c, r0);
    tc::tmem_ld16_nowait(taddr + kColV + c + 16, r1);
    tc::tmem_wait_ld();
    float dz[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const float x = __fadd_rn(__uint_as_float(q < 16 ? r0[q] : r1[q - 16]), relr[c + q]);
      dz[q] = sc == 0.f ? 0.f : (L2 ? __fmul_rn(x, sc) : (x > 0.f ? sc : (x < 0.f ? -sc : 0.f)));
    }
#pragma unroll
    for (int q = 0; q < 32; q += 8) {
      const int fl = (m >> 2) & 1;
      const float4 a = make_float4(dz[q], dz[q + 1], dz[q + 2], dz[q + 3]);
      const float4 b = make_float4(dz[q + 4], dz[q + 5], dz[q + 6], dz[q + 7]);
      const int ua = tile_unit(m, (c + q) >> 2), ub = tile_unit(m, (c + q + 4) >> 2);
      *reinterpret_cast<float4*>(S.DZ + 4 * (fl ? ub : ua)) = f4sel(fl, b, a);
      *reinterpret_cast<float4*>(S.DZ + 4 * (fl ? ua : ub)) = f4sel(fl, a, b);
    }
    float lo[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) lo[q] = tc::tf32_trunc_lo(dz[q]);
    tc::tmem_st16(taddr + kColHi + c, dz);
    tc::tmem_st16(taddr + kColHi + c + 16, dz + 16);
    tc::tmem_st16(taddr + kColLo + c, lo);
    tc::tmem_st16(taddr + kColLo + c + 16, lo + 16);
    // transpose-reduce the 32 x 32 block: lane l ends with the column c + l sum
#pragma unroll
    for (int ww = 16; ww >= 1; ww >>= 1) {
      const bool upper = (lane & ww) != 0;
#pragma unroll
      for (int q = 0; q < ww; ++q) {
        const float send = upper ? dz[q] : dz[q + ww];
        const float keep = upper ? dz[q + ww] : dz[q];
        dz[q] = __fadd_rn(keep, __shfl_xor_sync(kFull, send, ww));
      }
    }
    S.colsum[w][c + lane] = dz[0];
  }
}

__device__ __forceinline__ uint32_t idesc128() { return tc::make_idesc_tf32(128, 128, 0, 0); }

// Relation-segment ordinal of tile t (tiles of a segment are contiguous).
__device__ __forceinline__ int run_of(const Args& a, uint32_t t) {
  uint32_t lo = 0, hi = a.tile_total[1];
  while (lo + 1 < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a.seg_tiles[mid] <= t) lo = mid;
    else hi = mid;
  }
  return static_cast<int>(lo);
}

// Row ids of tile t by one warp: lane l resolves pairs l and l + 32 (positive
// row = batch position; its negative is row B + position, same relation).
__device__ __forceinline__ void chase_rows(const Args& a, uint32_t t, int lane, int4* rows, float* rel, int* np_out) {
  const FwdArgs& f = a.f;
  const uint32_t sseg = __ldg(a.tile_seg + t), p0 = __ldg(a.tile_p0 + t);
  const uint32_t e0 = __ldg(a.seg_start + sseg), len = __ldg(a.seg_start + sseg + 1) - e0;
  const int64_t r = static_cast<int64_t>(__ldg(a.seg_col + sseg)) - f.N;
  const int np = static_cast<int>(min(static_cast<uint32_t>(kPairs), len / 2 - p0));
  int pos[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int kk = lane + 32 * q;
    pos[q] = kk < np ? static_cast<int>(__ldg(a.ent_val + e0 + p0 + kk) & 0x7fffffffu) : -1;
  }
  const float4 rv = lane < (f.dr >> 2)  // d_r-wide relation row, zero-padded to kD
                        ? __ldg(reinterpret_cast<const float4*>(f.X + f.N * static_cast<int64_t>(f.de) + r * f.dr) + lane)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int kk = lane + 32 * q;
    int4 pr = make_int4(0, 0, -1, 0), ng = make_int4(0, 0, -1, 0);
    if (pos[q] >= 0) {
      int h, tt, nh, nt;
      if (f.pair_ht) {
        const int4 x = __ldg(f.pair_ht + pos[q]);
        h = x.x, tt = x.y, nh = x.z, nt = x.w;
      } else {
        const int id = __ldg(f.order + pos[q]);
        h = __ldg(f.H + id), tt = __ldg(f.T + id), nh = __ldg(f.NH + id), nt = __ldg(f.NT + id);
      }
      pr = make_int4(h, tt, pos[q], 0);
      ng = make_int4(nh, nt, pos[q] + f.B, 0);
    }
    rows[kk] = pr;
    rows[64 + kk] = ng;
  }
  reinterpret_cast<float4*>(rel)[lane] = rv;
  if (lane == 0) *np_out = np;
}

// CTAs that take tiles: the fewest giving the same longest range as all G, so
// the spare SMs stay free for the graph's side branches (a persistent CTA that
// finds its SM held by a long plan-branch block would start late and hold up
// the batch). Training kernel and apply agree on it, both from T.
__device__ __forceinline__ uint32_t working_ctas(uint32_t T, uint32_t G) {
  if (T == 0) return G;
  const uint32_t per = (T + G - 1) / G;
  return (T + per - 1) / per;
}

template <bool L2>
__global__ void __launch_bounds__(kThreads, 1)
    transr_train_tc_kernel(const Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const FwdArgs& f = a.f;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool alive = f.err[0] == 0;
  const bool tr = g_trace_on == f.batch + 1;  // trace one chosen minibatch
  if (f.stamp_start && blockIdx.x == 0 && tid == 0) stamp_now(f.stamp_start);  // the batch's first kernel (tiles planned)
  auto trace = [&](uint32_t it, int ev) { trace_ev(tr, it, ev); };
  // globaltimer stamps (comparable across SMs) in the last tile slot: 15 CTA start,
  // 14 first tile's rows seen by the producers, 13 loops done, 12 loss written
  auto gtrace = [&](int ev) {
    if (tr && blockIdx.x < kTrCtas) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      g_trace[(blockIdx.x * kTrTiles + kTrTiles - 1) * kTrEvents + ev] = g;
    }
  };
  if (tid == 0) gtrace(15);

  if (warp == 0) tc::tmem_alloc(&S.tmem_base, 512);
  if (f.de < kD)  // row tiles narrower than 128: the gather never writes columns >= d_e, keep them zero
    for (int i = tid; i < kRows * (kD - f.de) / 4; i += kThreads) {
      const int r = i / ((kD - f.de) / 4), c4 = (f.de >> 2) + i % ((kD - f.de) / 4);
      reinterpret_cast<float4*>(S.U)[tile_unit(r, c4)] = make_float4(0.f, 0.f, 0.f, 0.f);
      reinterpret_cast<float4*>(S.DZ)[tile_unit(r, c4)] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  if (tid == 0) {
    tc::mbar_init(&S.g_full, 32 * kGatherWarps);
    for (int q = 0; q < 4; ++q) tc::mbar_init(&S.u_q[q], 256);
    tc::mbar_init(&S.v_full, 1);
    tc::mbar_init(&S.dz_full, kDzSplit < kD ? 256 : 128);
    tc::mbar_init(&S.sc_full, 128);
    tc::mbar_init(&S.g2_done, 1);
    tc::mbar_init(&S.du_empty, 128);
    tc::mbar_init(&S.dm_full, 1);
    tc::mbar_init(&S.dm_empty, 128);
    for (int i = 0; i < kG3Slots; ++i) {
      tc::mbar_init(&S.g3_full[i], 128);
      tc::mbar_init(&S.g3_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&S.rows_full[i], 1);
      tc::mbar_init(&S.rows_empty[i], 128);
    }
    for (int i = 0; i < kRows / 8; ++i) tc::mbar_init(&S.stg[i], 1);
    for (int i = 0; i < kRing; ++i) {
      tc::mbar_init(&S.ring_full[i], 1);
      tc::mbar_init(&S.ring_empty[i], 1);
    }
    tc::fence_barrier_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = S.tmem_base;
  if ((tc::smem_u32(S.U) & 1023u) != 0) __trap();  // SWIZZLE_128B atoms need 1 KB alignment

  const uint32_t T = alive ? a.tile_total[0] : 0u;
  const uint32_t G = working_ctas(T, gridDim.x);
  const uint32_t b = blockIdx.x < G ? blockIdx.x : G;  // CTAs past G take no tile
  const uint32_t t0 = static_cast<uint32_t>((static_cast<uint64_t>(T) * b) / G);
  const uint32_t t1 = blockIdx.x < G ? static_cast<uint32_t>((static_cast<uint64_t>(T) * (b + 1)) / G) : t0;
  const uint32_t ntile = t1 - t0;

  float lsum = 0.f;
  uint32_t pend = 0;

  if (warp < 4) {
    // ------------------------------------------------------------ epilogue
    const int m = tid;  // row == TMEM lane
    const uint32_t lane_addr = static_cast<uint32_t>(warp * 32) << 16;
    float dr_acc = 0.f;
    int run = -1;
    uint32_t nrun = 0;
    for (uint32_t it = 0; it < ntile; ++it) {
      const uint32_t t = t0 + it;
      const int k = run_of(a, t);
      if (run >= 0 && k != run) ++nrun;
      run = k;
      const bool last_of_run = (t + 1 == t1) || (a.seg_tiles[k + 1] <= t + 1);
      const int buf = it & 1;
      tc::mbar_wait(&S.rows_full[buf], (it >> 1) & 1);  // tile metadata (rows, rel, np)
      tc::mbar_wait(&S.u_q[3], it & 1);
      tc::mbar_wait(&S.v_full, it & 1);
      tc::fence_after();
      if (m == 0) trace(it, 11);
      const float* relr = S.rel[buf];
      const int np = S.np[buf];
      const int row2 = S.rows[buf][m].z;
      // pass 1: v = V + r, reference-order squared_sum / abs_sum (norms.hpp:19-55)
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll 1
      for (int c = 0; c < kD; c += 32) {
        uint32_t r0[16], r1[16];
        tc::tmem_ld16_nowait(tbase + lane_addr + kColV + c, r0);
        tc::tmem_ld16_nowait(tbase + lane_addr + kColV + c + 16, r1);
        tc::tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 32; q += 4) {
          const uint32_t* rr = q < 16 ? r0 + q : r1 + (q - 16);
          s0 = __fadd_rn(s0, norm_term<L2>(__fadd_rn(__uint_as_float(rr[0]), relr[c + q])));
          s1 = __fadd_rn(s1, norm_term<L2>(__fadd_rn(__uint_as_float(rr[1]), relr[c + q + 1])));
          s2 = __fadd_rn(s2, norm_term<L2>(__fadd_rn(__uint_as_float(rr[2]), relr[c + q + 2])));
          s3 = __fadd_rn(s3, norm_term<L2>(__fadd_rn(__uint_as_float(rr[3]), relr[c + q + 3])));
        }
      }
      const float ssum = __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
      // terms are >= 0 or NaN: a finite sum proves every element of v finite;
      // otherwise the warp rescans V (tcgen05.ld is warp-collective)
      bool bad = false;
      if (__any_sync(kFull, nonfinite(ssum))) {
#pragma unroll 1
        for (int c = 0; c < kD; c += 16) {
          uint32_t r0[16];
          tc::tmem_ld16_nowait(tbase + lane_addr + kColV + c, r0);
          tc::tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 16; ++q) bad |= nonfinite(__fadd_rn(__uint_as_float(r0[q]), relr[c + q]));
        }
      }
      S.rs[m] = L2 ? __fsqrt_rn(ssum) : ssum;
      if (bad && row2 >= 0) pend |= kPendEntity;
      tc::named_sync(1, 128);
      // pair hinge (training.cpp:73-94): term = margin + E_pos - E_neg, active iff > 0
      const int kk = m & 63;
      const bool valid = kk < np;
      float term = 0.f;
      if (valid) term = __fsub_rn(__fadd_rn(f.margin, S.rs[kk]), S.rs[64 + kk]);
      const bool active = valid && term > 0.f;
      const float up = active ? (m < 64 ? f.unit : -f.unit) : 0.f;
      const float sc = up == 0.f ? 0.f : (L2 ? __fdiv_rn(up, __fsqrt_rn(__fadd_rn(ssum, kNormEpsF))) : up);
      // entity pass (kTileSlotRows): scal carries the dU row's tile slot + 1, 0 when inactive
      if (row2 >= 0) reinterpret_cast<uint32_t*>(f.scal)[row2] = active ? (t * kRows + static_cast<uint32_t>(m) + 1u) : 0u;
      {  // tile loss: positive rows, deterministic tree
        float v = (m < 64 && active) ? term : 0.f;
        if (warp < 2) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_down_sync(kFull, v, o));
          if (lane == 0) S.tl[warp] = v;
        }
      }
      // pass 2 (columns [0, kDzSplit); the producer warps take the rest)
      S.sc[m] = sc;
      if (kDzSplit < kD) tc::mbar_arrive(&S.sc_full);
      dz_pass<L2>(S, tbase + lane_addr, m, warp, sc, relr, 0, kDzSplit);
      tc::tmem_wait_st();
      tc::fence_before();
      tc::fence_async_shared();
      tc::mbar_arrive(&S.dz_full);
      if (m == 0) trace(it, 12);
      tc::mbar_wait(&S.dz_full, it & 1);  // every DZ row and column (and column sum) is written
      if (kStageStep == 2)  // the odd GEMM3 slots
        for (int s3 = 1; s3 < kG3PerTile; s3 += 2) stage_slot(S, it, s3, m);
      dr_acc = __fadd_rn(dr_acc, __fadd_rn(__fadd_rn(S.colsum[0][m], S.colsum[1][m]),
                                           __fadd_rn(S.colsum[2][m], S.colsum[3][m])));
      if (m == 0) lsum = __fadd_rn(lsum, __fadd_rn(S.tl[0], S.tl[1]));
      if (last_of_run) {  // flush the run's dM (lane = output row i) and sum(dz)
        tc::mbar_wait(&S.dm_full, nrun & 1);
        tc::fence_after();
        const uint32_t slot = blockIdx.x + static_cast<uint32_t>(k);
        float* dst = a.dm_part + static_cast<size_t>(slot) * kD * kD + static_cast<size_t>(m) * kD;
#pragma unroll 1
        for (int c = 0; c < kD; c += 32) {
          uint32_t r0[16], r1[16];
          tc::tmem_ld16_nowait(tbase + lane_addr + kColDM + c, r0);
          tc::tmem_ld16_nowait(tbase + lane_addr + kColDM + c + 16, r1);
          tc::tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 16; q += 4) {
            *reinterpret_cast<float4*>(dst + c + q) = make_float4(__uint_as_float(r0[q]), __uint_as_float(r0[q + 1]),
                                                                  __uint_as_float(r0[q + 2]), __uint_as_float(r0[q + 3]));
            *reinterpret_cast<float4*>(dst + c + 16 + q) = make_float4(
                __uint_as_float(r1[q]), __uint_as_float(r1[q + 1]), __uint_as_float(r1[q + 2]), __uint_as_float(r1[q + 3]));
          }
        }
        a.dr_part[static_cast<size_t>(slot) * kD + m] = dr_acc;
        dr_acc = 0.f;
        tc::fence_before();
        tc::mbar_arrive(&S.dm_empty);
      }
      // dU drain in tile-blocked order (kTileSlotRows): kDuGroup-float groups,
      // thread = row, 32-byte stores
      tc::mbar_wait(&S.g2_done, it & 1);
      tc::fence_after();
      if (m == 0) trace(it, 13);
      float* dst = f.res_u + static_cast<size_t>(t) * kRows * kD + static_cast<size_t>(m) * kDuGroup;
#pragma unroll 1
      for (int c = 0; c < kD; c += 32) {
        uint32_t r[32];
        tc::tmem_ld16_nowait(tbase + lane_addr + kColDU + c, r);
        tc::tmem_ld16_nowait(tbase + lane_addr + kColDU + c + 16, r + 16);
        tc::tmem_wait_ld();
#ifdef SKG_TR_NO_DRAIN
        if (false) {
#else
        if (active) {
#endif
#pragma unroll
          for (int q = 0; q < 32; q += 8)
            st_global_v8(dst + ((c + q) / kDuGroup) * (kRows * kDuGroup) + (c + q) % kDuGroup, r + q);
        }
      }
      tc::fence_before();
      tc::mbar_arrive(&S.du_empty);
      tc::mbar_arrive(&S.rows_empty[buf]);
      if (m == 0) trace(it, 14);
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------ producers
    const int p = tid - 128;   // row p == TMEM lane p (warp quadrant = warp % 4)
    const int pw = warp - 4;
    const uint32_t lane_addr = static_cast<uint32_t>(pw * 32) << 16;
    for (uint32_t it = 0; it < ntile; ++it) {
      const int buf = it & 1;
      tc::mbar_wait(&S.rows_full[buf], (it >> 1) & 1);
      if (p == 0) trace(it, 0);
      if (p == 0 && it == 0) gtrace(14);
      const int4* rows = S.rows[buf];
      tc::mbar_wait(&S.g_full, it & 1);  // head rows in sU, tail rows in sDZ
      if (p == 0) trace(it, 1);
      // U = h - t in place (row p), hi / lo -> TMEM once GEMM2 of the previous
      // tile has consumed DZ hi / lo
      if (it > 0) {
        tc::mbar_wait(&S.g2_done, (it - 1) & 1);
        tc::fence_after();
      }
      if (p == 0) trace(it, 15);
      // U by K quarters (this group: columns [32 q, 32 q + 16), the gather warps the other
      // 16), each quarter released to GEMM1 as soon as it is in TMEM
#pragma unroll 1
      for (int q = 0; q < 4; ++q) {
        compute_u(S, tbase + lane_addr, p, rows[p].z >= 0, 32 * q, 32 * q + 16, f.de);
        tc::tmem_wait_st();
        tc::fence_before();
        tc::mbar_arrive(&S.u_q[q]);
      }
      if (p == 0) trace(it, 2);
      if (kDzSplit < kD) {  // pass 2 of the epilogue on columns [kDzSplit, kD) of this warp's TMEM lanes
        tc::mbar_wait(&S.sc_full, it & 1);
        tc::fence_after();
        dz_pass<L2>(S, tbase + lane_addr, p, pw, S.sc[p], S.rel[buf], kDzSplit, kD);
        tc::tmem_wait_st();
        tc::fence_before();
        tc::fence_async_shared();
        tc::mbar_arrive(&S.dz_full);
      }
      // GEMM3 staging (even slots; the epilogue warps stage the odd ones)
      tc::mbar_wait(&S.dz_full, it & 1);
      if (p == 0) trace(it, 3);
      for (int s3 = 0; s3 < kG3PerTile; s3 += kStageStep) stage_slot(S, it, s3, p);
      if (p == 0) trace(it, 4);
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issue
    const uint32_t id = idesc128();
    const uint32_t id3 = tc::make_idesc_tf32(128, 128, 1, 1);  // GEMM3: both operands MN-major
    uint32_t rn = 0, g3n = 0, nrun = 0;
    int run = -1;
    for (uint32_t it = 0; it < ntile; ++it) {
      const uint32_t t = t0 + it;
      const int k = run_of(a, t);
      const bool first_of_run = k != run;
      if (run >= 0 && first_of_run) ++nrun;
      run = k;
      const bool last_of_run = (t + 1 == t1) || (a.seg_tiles[k + 1] <= t + 1);
      if (it > 0) tc::mbar_wait(&S.du_empty, (it - 1) & 1);  // V shares columns with the drained dU
      tc::mbar_wait(&S.u_q[0], it & 1);
      tc::fence_after();
      trace(it, 5);
      // GEMM1: V = U M_r^T, K quarter by K quarter as U's columns land in TMEM
      for (int c = 0; c < kChunksPerGemm; ++c, ++rn) {
        if (c > 0 && (c & 1) == 0) {
          tc::mbar_wait(&S.u_q[c >> 1], it & 1);
          tc::fence_after();
        }
        const int s = rn % kRing;
        tc::mbar_wait(&S.ring_full[s], (rn / kRing) & 1);
        tc::fence_after();
        const uint32_t bh = tc::smem_u32(S.ring[s]), bl = bh + kChunkFloats * 4;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int ks = c * 2 + kk;
          const uint64_t bhd = tc::make_desc(bh + kk * 256, kChLBO, kChSBO);
          const uint64_t bld = tc::make_desc(bl + kk * 256, kChLBO, kChSBO);
          tc::mma_ts_elect(tbase + kColV, tbase + kColHi + ks * 8, bhd, id, ks > 0 ? 1u : 0u);
          tc::mma_ts_elect(tbase + kColV, tbase + kColHi + ks * 8, bld, id, 1u);
          tc::mma_ts_elect(tbase + kColV, tbase + kColLo + ks * 8, bhd, id, 1u);
        }
        tc::commit_elect(&S.ring_empty[s]);
      }
      tc::commit_elect(&S.v_full);
      trace(it, 6);
      // GEMM3: dM += DZ^T U over the staged 8-row slots
      if (first_of_run && nrun > 0) {
        tc::mbar_wait(&S.dm_empty, (nrun - 1) & 1);
        tc::fence_after();
      }
      // GEMM3 over the 16 staged slots first: each slot's commit releases its
      // row group of sU / sDZ to the next tile's gather, so the gather runs
      // under GEMM2 (dU = DZ M_r; DZ hi / lo from TMEM), issued after it.
      tc::mbar_wait(&S.dz_full, it & 1);
      tc::fence_after();
      trace(it, 9);
      auto gemm2_chunk = [&](int c) {
        const int s = rn % kRing;
        tc::mbar_wait(&S.ring_full[s], (rn / kRing) & 1);
        tc::fence_after();
        const uint32_t bh = tc::smem_u32(S.ring[s]), bl = bh + kChunkFloats * 4;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int ks = c * 2 + kk;
          const uint64_t bhd = tc::make_desc(bh + kk * 256, kChLBO, kChSBO);
          const uint64_t bld = tc::make_desc(bl + kk * 256, kChLBO, kChSBO);
          tc::mma_ts_elect(tbase + kColDU, tbase + kColHi + ks * 8, bhd, id, ks > 0 ? 1u : 0u);
          tc::mma_ts_elect(tbase + kColDU, tbase + kColHi + ks * 8, bld, id, 1u);
          tc::mma_ts_elect(tbase + kColDU, tbase + kColLo + ks * 8, bhd, id, 1u);
        }
        tc::commit_elect(&S.ring_empty[s]);
        ++rn;
      };
      for (int s3 = 0; s3 < kG3PerTile; ++s3, ++g3n) {
        const int slot = g3n % kG3Slots;
        tc::mbar_wait(&S.g3_full[slot], (g3n / kG3Slots) & 1);
        tc::fence_after();
        if (s3 == 0) trace(it, 7);
        const uint32_t roff = static_cast<uint32_t>(s3 * kG3Rows * 128);  // the slot's rows in sDZ / sU
        const uint64_t ahi = tc::make_desc_sw128_32b(tc::smem_u32(S.DZ) + roff, kTileLBO, kSBO32);
        const uint64_t bhi = tc::make_desc_sw128_32b(tc::smem_u32(S.U) + roff, kTileLBO, kSBO32);
        const uint64_t alo = tc::make_desc_sw128_32b(tc::smem_u32(S.g3[slot][0]), kG3LBO, kSBO32);
        const uint64_t blo = tc::make_desc_sw128_32b(tc::smem_u32(S.g3[slot][1]), kG3LBO, kSBO32);
        tc::mma_ss_elect(tbase + kColDM, ahi, bhi, id3, (first_of_run && s3 == 0) ? 0u : 1u);
        tc::mma_ss_elect(tbase + kColDM, ahi, blo, id3, 1u);
        tc::mma_ss_elect(tbase + kColDM, alo, bhi, id3, 1u);
        tc::commit_elect(&S.g3_empty[slot]);
        tc::commit_elect(&S.stg[s3]);  // row group s3 of sU / sDZ read: the gather may refill it
        if (s3 == kG3PerTile - 1 && last_of_run) tc::commit_elect(&S.dm_full);
#ifndef SKG_TR_G2_AFTER
        if (s3 & 1) gemm2_chunk(s3 >> 1);
#endif
      }
#ifdef SKG_TR_G2_AFTER
      for (int c = 0; c < kChunksPerGemm; ++c) gemm2_chunk(c);
#endif
      trace(it, 8);
      tc::commit_elect(&S.g2_done);
      trace(it, 10);
    }
  } else if (warp == kRowWarp) {
    // ------------------------------------------------------------ row-id chase
    for (uint32_t it = 0; it < ntile; ++it) {
      const int buf = it & 1;
      if (it >= 2) tc::mbar_wait(&S.rows_empty[buf], ((it >> 1) - 1) & 1);
      chase_rows(a, t0 + it, lane, S.rows[buf], S.rel[buf], &S.np[buf]);
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&S.rows_full[buf]);
#ifndef SKG_TR_NO_PREFETCH
      // pull the tile's head / tail rows into L2 now, a tile or more before
      // the gather warp copies them (they miss L2 about half the time at C4:
      // the table and the per-batch dU rows together exceed it)
#pragma unroll 4
      for (int k = lane; k < 4 * kRows; k += 32) {
        const int4 rw = S.rows[buf][k >> 2];
        const int hv = (k >> 1) & 1;
        if (hv * 64 < f.de) {
          const float* row = f.X + static_cast<size_t>((k & 1) ? rw.y : rw.x) * f.de + hv * 64;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(row));
          if (hv * 64 + 32 < f.de) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + 32));
        }
      }
#endif
    }
  } else if (warp >= kGatherWarp) {
    // ------------------------------------------------------------ row gather
    // 16-byte cp.async per lane (lane = chunk of a 512-byte row): head rows
    // into sU, tail rows into sDZ at tile_unit; one warp keeps a tile's 256
    // rows in flight without registers. (TMA tile::gather4 of 128-byte boxes
    // measured ~16 cycles per box row per SM here, too slow to hide.)
    const int de = f.de, de4 = de >> 2;
    auto gather8 = [&](const int4* rows, int r0) {  // rows r0 .. r0 + 7, head and tail
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int4 rw = rows[r0 + q];
        if (lane < de4) {  // d_e-wide rows; U's columns >= d_e are kept zero (compute_u)
          tc::cp_async16(S.U + 4 * tile_unit(r0 + q, lane), f.X + static_cast<size_t>(rw.x) * de + 4 * lane);
          tc::cp_async16(S.DZ + 4 * tile_unit(r0 + q, lane), f.X + static_cast<size_t>(rw.y) * de + 4 * lane);
        }
      }
    };
    for (uint32_t it = 0; it < ntile; ++it) {
      const int buf = it & 1;
      tc::mbar_wait(&S.rows_full[buf], (it >> 1) & 1);
      const int4* rows = S.rows[buf];
#ifdef SKG_TR_GATHER_BULK
      if (it > 0) tc::mbar_wait(&S.stg[kG3PerTile - 1], (it - 1) & 1);
#endif
#pragma unroll 1
      for (int s3 = warp - kGatherWarp; s3 < kG3PerTile; s3 += kGatherWarps) {
        // tile it's rows go into the row groups GEMM3 of tile it - 1 has consumed
        if (it > 0) tc::mbar_wait(&S.stg[s3], (it - 1) & 1);
        gather8(rows, s3 * 8);
      }
      tc::cp_async_mbar_arrive(&S.g_full);
      {  // columns [32 q + 16, 32 q + 32) of U for the rows of this warp's TMEM lane quadrant
        const int q4 = warp & 3;
        const int row = q4 * 32 + lane;
        tc::mbar_wait(&S.g_full, it & 1);
        if (it > 0) {
          tc::mbar_wait(&S.g2_done, (it - 1) & 1);
          tc::fence_after();
        }
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {
          compute_u(S, tbase + (static_cast<uint32_t>(q4 * 32) << 16), row, rows[row].z >= 0, 32 * q + 16,
                    32 * q + 32, f.de);
          tc::tmem_wait_st();
          tc::fence_before();
          tc::mbar_arrive(&S.u_q[q]);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ ring loader
    uint32_t rn = 0;
    for (uint32_t it = 0; it < ntile; ++it) {
      const uint32_t t = t0 + it;
      const int64_t r = static_cast<int64_t>(__ldg(a.seg_col + __ldg(a.tile_seg + t))) - f.N;
      for (int layout = 0; layout < 2; ++layout)
        for (int c = 0; c < kChunksPerGemm; ++c, ++rn) {
          const int s = rn % kRing;
          if (rn >= kRing) tc::mbar_wait(&S.ring_empty[s], ((rn / kRing) - 1) & 1);
          if (lane == 0) {
            const float* src = a.mr + r * kMrFloatsPerRel + static_cast<int64_t>(layout * kChunksPerGemm + c) * 2 * kChunkFloats;
            tc::mbar_arrive_expect_tx(&S.ring_full[s], kChunkBytes);
            tc::bulk_g2s(S.ring[s], src, kChunkBytes, &S.ring_full[s]);
          }
          __syncwarp();
        }
    }
  }

  // ---- teardown, loss: one partial per CTA, the last CTA finalizes (tile order)
  tc::fence_before();
  __syncthreads();
  if (tid == 0) gtrace(13);
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
  if (warp < 4) {
    pend = __reduce_or_sync(kFull, pend);
    if (lane == 0 && pend) {
      atomicOr(&f.err[3], pend);
      __threadfence();
    }
  }
  if (!alive) return;
  if (tid == 0) {
    f.block_partial[blockIdx.x] = lsum;
    S.last = ticket_acq_rel(f.counter) == gridDim.x - 1;
  }
  __syncthreads();
  if (S.last && warp == 0) {
    float acc = 0.f;
    for (int b = lane; b < static_cast<int>(gridDim.x); b += 32) acc = __fadd_rn(acc, f.block_partial[b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_down_sync(kFull, acc, o));
    if (lane == 0) {
      const float loss = __fdiv_rn(acc, f.loss_div > 0.f ? f.loss_div : static_cast<float>(f.B));
      f.batch_loss[f.batch] = loss;
      if (f.stamp_end) stamp_now(f.stamp_end);
      gtrace(12);
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

// Per relation: both K-major operand views of M_r in 16-wide K chunks, split
// hi (rna tf32) / lo, laid out exactly as the ring slots are read.
//   layout 0 (GEMM1 B): n = output row i, k = j;  layout 1 (GEMM2 B): n = j, k = i.
// M_r is d_r x d_e (models.hpp:23-29); entries outside it are zero, so the
// padded GEMMs give zero V columns >= d_r and zero dU columns >= d_e.
__global__ void transr_train_prep_kernel(const float* __restrict__ proj, float* __restrict__ out, int dr, int de) {
  const int r = blockIdx.x, lc = blockIdx.y;  // lc = layout * 8 + chunk
  const int layout = lc >> 3, k0 = (lc & 7) * kChunkK;
  const float* M = proj + static_cast<int64_t>(r) * dr * de;
  float* hi = out + r * kMrFloatsPerRel + static_cast<int64_t>(lc) * 2 * kChunkFloats;
  float* lo = hi + kChunkFloats;
  for (int i = threadIdx.x; i < kChunkFloats; i += blockDim.x) {
    int n, kk;
    float x;
    if (layout == 0) {  // M[n][k0 + kk]: 16 consecutive floats per row
      n = i >> 4;
      kk = i & 15;
      x = n < dr && k0 + kk < de ? M[n * de + k0 + kk] : 0.f;
    } else {            // M[k0 + kk][n]: coalesced along n
      kk = i >> 7;
      n = i & 127;
      x = k0 + kk < dr && n < de ? M[(k0 + kk) * de + n] : 0.f;
    }
    float h, l;
    tc::split_tf32(x, h, l);
    const int o = (((n & 7) + (n >> 3) * 32 + (kk >> 2) * 8) << 2) + (kk & 3);
    hi[o] = h;
    lo[o] = l;
  }
}

// Per relation segment k of the batch: sum the (CTA, relation run) partials
// j + k in CTA order (the partition transr_train_tc_kernel used), SGD on M_r
// and the relation row, and refresh M_r's pre-split ring chunks so the next
// minibatch needs no separate split pass.
__global__ void transr_train_apply_kernel(const uint32_t* __restrict__ tile_total,
                                          const uint32_t* __restrict__ seg_tiles,
                                          const uint32_t* __restrict__ tile_seg, const uint32_t* __restrict__ seg_col,
                                          int64_t N, int G, const float* __restrict__ dm_part,
                                          const float* __restrict__ dr_part, float* __restrict__ proj,
                                          float* __restrict__ rel, const float* __restrict__ lr,
                                          const uint32_t* __restrict__ err, float* __restrict__ mr, int sink, int dr,
                                          int de) {
  if (err[0] != 0) return;
  const uint32_t k = blockIdx.x;
  if (k >= tile_total[1]) return;
  const uint32_t T = tile_total[0];
  G = static_cast<int>(working_ctas(T, static_cast<uint32_t>(G)));
  const uint32_t lo = seg_tiles[k], hi = seg_tiles[k + 1];
  if (hi <= lo) return;
  const int64_t r = static_cast<int64_t>(seg_col[tile_seg[lo]]) - N;
  const float step = *lr;
  __shared__ int jl[1024];
  __shared__ int nj;
  if (threadIdx.x < 32) {  // CTAs j whose tile range [T j / G, T (j+1) / G) meets [lo, hi), in order
    int c = 0;
    for (int j0 = 0; j0 < G && j0 < 1024; j0 += 32) {
      const int j = j0 + static_cast<int>(threadIdx.x);
      bool o = false;
      if (j < G && j < 1024) {
        const uint32_t a0 = static_cast<uint32_t>((static_cast<uint64_t>(T) * j) / G);
        const uint32_t a1 = static_cast<uint32_t>((static_cast<uint64_t>(T) * (j + 1)) / G);
        o = a0 < a1 && a1 > lo && a0 < hi;
      }
      const unsigned m = __ballot_sync(kFull, o);
      if (o) jl[c + __popc(m & lanemask_lt())] = j;
      c += __popc(m);
    }
    if (threadIdx.x == 0) nj = c;
  }
  __syncthreads();
  float* mrr = mr + r * kMrFloatsPerRel;
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < kD * kD + kD; i += gridDim.y * blockDim.x) {
    const bool pm = i < kD * kD;
    float g = 0.f;
    int q = 0;
    for (; q + 4 <= nj; q += 4) {  // four independent loads in flight, added in order
      float v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const size_t slot = static_cast<size_t>(jl[q + e]) + k;
        v[e] = pm ? __ldcg(dm_part + slot * kD * kD + i) : __ldcg(dr_part + slot * kD + (i - kD * kD));
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) g = __fadd_rn(g, v[e]);
    }
    for (; q < nj; ++q) {
      const size_t slot = static_cast<size_t>(jl[q]) + k;
      g = __fadd_rn(g, pm ? __ldcg(dm_part + slot * kD * kD + i) : __ldcg(dr_part + slot * kD + (i - kD * kD)));
    }
    const int a = i / kD, b = i - a * kD;  // M_r element (a, b), or relation column i - kD * kD
    if (pm ? (a >= dr || b >= de) : (i - kD * kD >= dr)) continue;  // padding of a narrower M_r / relation row
    float* p = pm ? proj + r * dr * de + a * de + b : rel + r * dr + (i - kD * kD);
    if (sink) {  // data parallel: this rank's gradient, one dense step after the all-reduce
      *p = g;
      continue;
    }
    const float nv = __fsub_rn(*p, __fmul_rn(step, g));
    *p = nv;
    if (pm) {  // element (row a = output dim, col b = entity dim) of M_r into both ring layouts
      float h, l;
      tc::split_tf32(nv, h, l);
      float* c0 = mrr + static_cast<int64_t>(b / kChunkK) * 2 * kChunkFloats;                   // layout 0: n = a, k = b
      float* c1 = mrr + static_cast<int64_t>(kChunksPerGemm + a / kChunkK) * 2 * kChunkFloats;  // layout 1: n = b, k = a
      const int kb = b % kChunkK, ka = a % kChunkK;
      const int o0 = (((a & 7) + (a >> 3) * 32 + (kb >> 2) * 8) << 2) + (kb & 3);
      const int o1 = (((b & 7) + (b >> 3) * 32 + (ka >> 2) * 8) << 2) + (ka & 3);
      c0[o0] = h;
      c0[kChunkFloats + o0] = l;
      c1[o1] = h;
      c1[kChunkFloats + o1] = l;
    }
  }
}

}  // namespace

int64_t transr_train_tc_mr_floats(int64_t R) { return R * kMrFloatsPerRel; }

int64_t transr_trace(int enable, unsigned long long* out, int64_t cap) {
  SKG_CUDA(cudaMemcpyToSymbol(g_trace_on, &enable, sizeof(int)));
  const int64_t n = static_cast<int64_t>(kTrCtas) * kTrTiles * kTrEvents;
  if (enable) {
    static const unsigned long long zeros[kTrCtas * kTrTiles * kTrEvents] = {};
    SKG_CUDA(cudaMemcpyToSymbol(g_trace, zeros, sizeof(zeros)));
  }
  if (out && cap >= n) SKG_CUDA(cudaMemcpyFromSymbol(out, g_trace, sizeof(unsigned long long) * n));
  return n;
}

// Training kernel widths: d_e, d_r multiples of 16 up to 128 (zero-padded tiles).
bool transr_train_tc_supported(int de, int dr) {
  return de >= 16 && dr >= 16 && de <= kD && dr <= kD && de % 16 == 0 && dr % 16 == 0;
}

void configure_transr_train_tc_kernels() {
  SKG_CUDA(cudaFuncSetAttribute(transr_train_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(Smem))));
  SKG_CUDA(cudaFuncSetAttribute(transr_train_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(Smem))));
}

void launch_transr_train_tc(bool l2, const FwdArgs& fa, const uint32_t* ent_val, const uint32_t* seg_start,
                            const uint32_t* seg_col, const uint32_t* tile_seg, const uint32_t* tile_p0,
                            const uint32_t* tile_total, const uint32_t* seg_tiles, float* dm_part, float* dr_part,
                            float* mr, int64_t R, int num_sms, cudaStream_t s, bool always_prep) {
  // the split M_r chunks are refreshed by every batch's apply; the first batch
  // of an epoch re-splits from proj (the store may have been replaced)
  if (fa.batch == 0 || always_prep) {
    transr_train_prep_kernel<<<dim3(static_cast<unsigned>(R), 2 * kChunksPerGemm), 256, 0, s>>>(fa.proj, mr, fa.dr,
                                                                                                 fa.de);
    count_launch();
  }
  Args a{};
  a.f = fa;
  a.ent_val = ent_val;
  a.seg_start = seg_start;
  a.seg_col = seg_col;
  a.tile_seg = tile_seg;
  a.tile_p0 = tile_p0;
  a.tile_total = tile_total;
  a.seg_tiles = seg_tiles;
  a.dm_part = dm_part;
  a.dr_part = dr_part;
  a.mr = mr;
  const size_t smem = sizeof(Smem);
  if (l2) transr_train_tc_kernel<true><<<num_sms, kThreads, smem, s>>>(a);
  else transr_train_tc_kernel<false><<<num_sms, kThreads, smem, s>>>(a);
  count_launch();
  SKG_LAUNCH_CHECK();
}

void launch_transr_train_apply(const uint32_t* tile_total, const uint32_t* seg_tiles, const uint32_t* tile_seg,
                               const uint32_t* seg_col, int64_t N, int G, const float* dm_part, const float* dr_part,
                               float* proj, float* rel, const float* lr, const uint32_t* err, float* mr, int64_t R,
                               cudaStream_t s, int sink, int dr, int de) {
  transr_train_apply_kernel<<<dim3(static_cast<unsigned>(R), SKG_APPLY_Y), 256, 0, s>>>(tile_total, seg_tiles, tile_seg, seg_col,
                                                                              N, G, dm_part, dr_part, proj, rel, lr,
                                                                              err, mr, sink, dr, de);
  count_launch();
  SKG_LAUNCH_CHECK();
}

}  // namespace skg
