// TransR projections on tcgen05 tensor cores (sm_100a), d_e = d_r = 128.
//
// Same data flow as transr.cu (relation-grouped tiles of 64 (pos, neg) pairs
// = 128 rows of one relation), but the three products run as 128x128x128
// MMAs with fp32 accumulators in TMEM:
//   GEMM1  V  = U M_r^T          A = U (K-major), B = M_r (K-major)
//   GEMM2  dU = DZ M_r           A = DZ, B = M_r^T (transposed while staging)
//   GEMM3  dM += DZ^T U          A = DZ^T, B = U^T (transposed while staging)
// All descriptors are K-major no-swizzle (the MN-major tf32 view is avoided).
// Precision: 3xTF32 (hi*hi + hi*lo + lo*hi, hi = rna-tf32(x), lo = x - hi),
// fp32-class results for the 1e-5 parity bar. Operands are kept in fp32 in
// shared memory (U, DZ) and split into hi/lo 32-wide K chunks staged in the
// canonical no-swizzle layouts (tc.cuh) right before each MMA group; one
// elected thread issues the MMAs and commits to an mbarrier.
//
// The TMEM lane = row mapping makes the epilogues thread-per-row: the score
// reduction of V runs in the reference's exact squared_sum order, and dM
// (lane = relation output row) is read back thread-per-row as well.
//
// CTAs are persistent: CTA j owns a contiguous range of the batch's tiles and
// accumulates dM (TMEM) and sum(dz) (registers) across consecutive tiles of the
// same relation, flushing one partial per (CTA, relation) run; the apply
// kernel sums runs in tile order (deterministic).
#include "common.cuh"
#include "ht.cuh"
#include "primitives.cuh"
#include "refmath.cuh"
#include "tc.cuh"

namespace skg {

namespace {

constexpr int kD = 128;        // d_e = d_r handled by this kernel
constexpr int kRows = 128;     // rows per tile
constexpr int kPairs = 64;
constexpr int kThreads = 256;  // 8 warps: warp w <-> TMEM lanes 32(w%4)..+31
constexpr int kEpi = 128;      // warps 0-3 run the row-per-thread epilogues
constexpr int kStride = kD + 4;
constexpr int kChunk = 32;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColV = 0, kColDU = 128, kColDM = 256;

enum Mode : int { kTrain = 0, kScore = 1, kPrep = 2 };

struct TcArgs {
  FwdArgs f;
  const uint32_t* ent_val;
  const uint32_t* seg_start;
  const uint32_t* seg_col;
  const uint32_t* tile_seg;
  const uint32_t* tile_p0;
  const uint32_t* tile_total;  // [0] tiles, [1] relation segments
  const uint32_t* seg_tiles;   // first tile of each relation segment
  float* dm_part;              // [slot][dr*de]
  float* dr_part;              // [slot][dr]
  const float* mr_chunks;      // per relation: [layout 2][chunk 4][hi,lo][128*32] pre-split M_r
};

// Per relation r, both K-major views of M_r, split hi/lo and laid out chunk by
// chunk exactly as the MMA reads them, so the projection CTAs fetch B operands
// with 16 KB bulk copies instead of re-splitting M_r for every tile.
//   layout 0 (GEMM1): rows n, k = c;   layout 1 (GEMM2): rows c, k = n.
constexpr int kChunkFloats = kD * kChunk;
constexpr int64_t kMrFloatsPerRel = 2 * 4 * 2 * kChunkFloats;
__global__ void transr_prep_mr_kernel(const float* __restrict__ proj, float* __restrict__ out) {
  const int r = blockIdx.x, lc = blockIdx.y;  // lc = layout * 4 + chunk
  const int layout = lc >> 2, kc = (lc & 3) * kChunk;
  const float* M = proj + static_cast<int64_t>(r) * kD * kD;
  float* hi = out + r * kMrFloatsPerRel + static_cast<int64_t>(lc) * 2 * kChunkFloats;
  float* lo = hi + kChunkFloats;
  for (int i = threadIdx.x; i < kChunkFloats; i += blockDim.x) {
    const int row = i / kChunk, k = i % kChunk;
    const float x = layout == 0 ? M[row * kD + kc + k] : M[(kc + k) * kD + row];
    float h, l;
    tc::split_tf32(x, h, l);
    const int o = tc::kmaj_off(row, k);
    hi[o] = h;
    lo[o] = l;
  }
}

struct Smem {
  float U[kRows * kStride];
  float DZ[kRows * kStride];
  float Ahi[kRows * kChunk], Alo[kRows * kChunk], Bhi[kD * kChunk], Blo[kD * kChunk];
};

__device__ __forceinline__ uint32_t idesc(int a_mn, int b_mn) { return tc::make_idesc_tf32(128, 128, a_mn, b_mn); }

// One 32-wide K chunk: 4 MMA k-steps x 3 products (hi*hi, hi*lo, lo*hi).
__device__ __forceinline__ void issue_chunk(const Smem& s, uint32_t tmem_d, bool a_mn, bool b_mn, bool first) {
  const uint32_t ahi = tc::smem_u32(s.Ahi), alo = tc::smem_u32(s.Alo);
  const uint32_t bhi = tc::smem_u32(s.Bhi), blo = tc::smem_u32(s.Blo);
  const uint32_t id = idesc(a_mn, b_mn);
  const uint32_t a_step = a_mn ? tc::kMnmajStepBytes : tc::kKmajStepBytes;
  const uint32_t b_step = b_mn ? tc::kMnmajStepBytes : tc::kKmajStepBytes;
  const uint32_t a_lbo = a_mn ? tc::kMnmajLBO : tc::kKmajLBO, a_sbo = a_mn ? tc::kMnmajSBO : tc::kKmajSBO;
  const uint32_t b_lbo = b_mn ? tc::kMnmajLBO : tc::kKmajLBO, b_sbo = b_mn ? tc::kMnmajSBO : tc::kKmajSBO;
#pragma unroll
  for (int st = 0; st < kChunk / 8; ++st) {
    const uint64_t dah = tc::make_desc(ahi + st * a_step, a_lbo, a_sbo);
    const uint64_t dal = tc::make_desc(alo + st * a_step, a_lbo, a_sbo);
    const uint64_t dbh = tc::make_desc(bhi + st * b_step, b_lbo, b_sbo);
    const uint64_t dbl = tc::make_desc(blo + st * b_step, b_lbo, b_sbo);
    tc::mma_tf32(tmem_d, dah, dbh, id, (first && st == 0) ? 0u : 1u);
    tc::mma_tf32(tmem_d, dah, dbl, id, 1u);
    tc::mma_tf32(tmem_d, dal, dbh, id, 1u);
  }
}

// Stage a K-major chunk (rows x 32) from a row-major fp32 source (row stride ld).
// Lane mapping: a warp covers one 8-row x 4-k core matrix (lane>>2 = row,
// lane&3 = k), so the 32 stores of a warp hit 32 distinct banks.
__device__ __forceinline__ void lane_rk(int i, int& r, int& k) {
  const int lane = i & 31, g = i >> 5;
  r = (g & 15) * 8 + (lane >> 2);
  k = (g >> 4) * 4 + (lane & 3);
}

__device__ __forceinline__ void stage_kmajor(float* hi, float* lo, const float* src, int ld, int k0, int rows,
                                             bool global_src) {
  for (int i = threadIdx.x; i < rows * kChunk; i += kThreads) {
    int r, k;
    lane_rk(i, r, k);
    const float x = global_src ? __ldg(src + static_cast<size_t>(r) * ld + k0 + k) : src[r * ld + k0 + k];
    float h, l;
    tc::split_tf32(x, h, l);
    const int o = tc::kmaj_off(r, k);
    hi[o] = h;
    lo[o] = l;
  }
}

// Stage a K-major chunk (128 rows x 32 k) from a source indexed [k][row]
// (row k0 + k, column row), row stride ld: the transposed operand views
// (M_r as [c][n] for dU, DZ^T and U^T for dM) are built here, so every MMA
// reads K-major descriptors.
__device__ __forceinline__ void stage_kmajor_t(float* hi, float* lo, const float* src, int ld, int k0,
                                               bool global_src) {
  for (int i = threadIdx.x; i < kD * kChunk; i += kThreads) {
    int r, k;
    lane_rk(i, r, k);
    const float x = global_src ? __ldg(src + static_cast<size_t>(k0 + k) * ld + r) : src[(k0 + k) * ld + r];
    float h, l;
    tc::split_tf32(x, h, l);
    const int o = tc::kmaj_off(r, k);
    hi[o] = h;
    lo[o] = l;
  }
}

__device__ __forceinline__ void mma_round(uint64_t* mbar, uint32_t& phase) {
  if (threadIdx.x == 0) tc::commit(mbar);
  tc::mbar_wait(mbar, phase);
  phase ^= 1u;
  tc::fence_after();
}

template <bool L2, int MODE>
__global__ void __launch_bounds__(kThreads, 1) transr_tc_kernel(const TcArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  __shared__ uint64_t mbar, bbar;
  __shared__ uint32_t tmem_base;
  __shared__ int rrow[kRows], rh[kRows], rt[kRows];
  __shared__ float rs[kRows], rsc[kRows];
  __shared__ float colsum[2][kD];
  __shared__ float relsh[kD];
  __shared__ float tile_loss_sh;
  const FwdArgs& f = a.f;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool alive = f.err[0] == 0;  // every CTA still joins the loss ticket below

  if (warp == 0) tc::tmem_alloc(&tmem_base, kTmemCols);
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    tc::mbar_init(&bbar, 1);
    tc::fence_barrier_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem_base;
  uint32_t bphase = 0;
  // B operand chunk (hi, lo) of M_r by bulk copy; issued before the A staging
  // so the copy overlaps it, awaited before the MMA.
  auto load_b = [&](int64_t rr, int layout, int chunk) {
    if (tid == 0) {
      const float* src = a.mr_chunks + rr * kMrFloatsPerRel + static_cast<int64_t>(layout * 4 + chunk) * 2 * kChunkFloats;
      tc::mbar_arrive_expect_tx(&bbar, 2 * kChunkFloats * sizeof(float));
      tc::bulk_g2s(S.Bhi, src, kChunkFloats * sizeof(float), &bbar);
      tc::bulk_g2s(S.Blo, src + kChunkFloats, kChunkFloats * sizeof(float), &bbar);
    }
  };
  auto wait_b = [&]() {
    tc::mbar_wait(&bbar, bphase);
    bphase ^= 1u;
  };
  const uint32_t lane_addr = static_cast<uint32_t>((warp & 3) * 32) << 16;
  const int qrow = (warp & 3) * 32 + lane;  // TMEM lane (row) of this thread
  const int half = warp >> 2;               // column half for the split epilogues
  uint32_t phase = 0;

  const uint32_t T = alive ? a.tile_total[0] : 0u;
  const uint32_t G = gridDim.x;
  const uint32_t t0 = static_cast<uint32_t>((static_cast<uint64_t>(T) * blockIdx.x) / G);
  const uint32_t t1 = static_cast<uint32_t>((static_cast<uint64_t>(T) * (blockIdx.x + 1)) / G);
  float lsum = 0.f;
  uint32_t pend = 0;
  int cur_k = -1;      // relation-segment ordinal of the open run
  float dr_acc = 0.f;  // thread n: running sum(dz) of the open run
  bool dm_first = true;
  const int de = kD, dr = kD;

  auto flush = [&](int k) {
    // slot index j + k: pieces of the (CTA range) x (relation run) partition
    const uint32_t slot = blockIdx.x + static_cast<uint32_t>(k);
    float* dst = a.dm_part + static_cast<size_t>(slot) * dr * de + static_cast<size_t>(qrow) * de;
    float v[16];
#pragma unroll 1
    for (int c = half * 64; c < half * 64 + 64; c += 16) {
      tc::tmem_ld16(tbase + lane_addr + kColDM + c, v);
#pragma unroll
      for (int q = 0; q < 16; q += 4) *reinterpret_cast<float4*>(dst + c + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
    }
    if (tid < kD) a.dr_part[static_cast<size_t>(slot) * dr + tid] = dr_acc;
    dr_acc = 0.f;
  };

  for (uint32_t t = t0; t < t1; ++t) {
    const uint32_t sseg = a.tile_seg[t], p0 = a.tile_p0[t];
    const uint32_t e0 = a.seg_start[sseg], len = a.seg_start[sseg + 1] - e0;
    const int64_t r = static_cast<int64_t>(a.seg_col[sseg]) - f.N;
    // relation-segment ordinal k: tiles of a segment are contiguous in the list
    int k = cur_k < 0 ? 0 : cur_k;
    if (cur_k < 0) {
      uint32_t lo = 0, hi = a.tile_total[1];
      while (lo + 1 < hi) {  // last k with seg_tiles[k] <= t
        const uint32_t mid = (lo + hi) >> 1;
        if (a.seg_tiles[mid] <= t) lo = mid;
        else hi = mid;
      }
      k = static_cast<int>(lo);
    } else {
      while (a.seg_tiles[k + 1] <= t) ++k;
    }
    if (MODE != kScore && cur_k >= 0 && k != cur_k) {
      flush(cur_k);
      dm_first = true;
    }
    cur_k = k;
    const uint32_t units = MODE == kTrain ? len / 2 : len;
    const int np = static_cast<int>(min(static_cast<uint32_t>(MODE == kTrain ? kPairs : kRows), units - p0));
    // ---- row ids (thread per row): incidence row, head and tail
    if (tid < kRows) {
      int row2 = -1, h = 0, tt = 0;
      if (MODE == kTrain) {
        const int kk = tid & 63;
        if (kk < np) row2 = static_cast<int>(a.ent_val[e0 + (tid < 64 ? 0 : units) + p0 + kk] & 0x7fffffffu);
      } else if (tid < np) {
        row2 = static_cast<int>(a.ent_val[e0 + p0 + tid] & 0x7fffffffu);
      }
      if (row2 >= 0) {
        if (MODE == kTrain) {
          const bool neg = row2 >= f.B;
          const int id = f.order[neg ? row2 - f.B : row2];
          h = neg ? f.NH[id] : f.H[id];
          tt = neg ? f.NT[id] : f.T[id];
        } else {
          h = f.H[row2];
          tt = f.T[row2];
        }
      }
      rrow[tid] = row2;
      rh[tid] = h;
      rt[tid] = tt;
      relsh[tid] = __ldg(f.X + f.N * static_cast<int64_t>(de) + r * dr + tid);
    }
    __syncthreads();
    // ---- U = h - t: each warp gathers 16 rows, 8 rows (16 x 16 B per lane) in flight
#pragma unroll 1
    for (int m0 = warp * 16; m0 < warp * 16 + 16; m0 += 8) {
      float4 xh[8], xt[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        xh[q] = __ldg(reinterpret_cast<const float4*>(f.X + static_cast<size_t>(rh[m0 + q]) * de) + lane);
        xt[q] = __ldg(reinterpret_cast<const float4*>(f.X + static_cast<size_t>(rt[m0 + q]) * de) + lane);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 u = rrow[m0 + q] >= 0 ? make_float4(__fsub_rn(xh[q].x, xt[q].x), __fsub_rn(xh[q].y, xt[q].y),
                                                          __fsub_rn(xh[q].z, xt[q].z), __fsub_rn(xh[q].w, xt[q].w))
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
        *reinterpret_cast<float4*>(S.U + (m0 + q) * kStride + 4 * lane) = u;
      }
    }
    __syncthreads();
    // ---- GEMM1: V = U M_r^T (K = de)
    for (int kc = 0; kc < de; kc += kChunk) {
      load_b(r, 0, kc / kChunk);
      stage_kmajor(S.Ahi, S.Alo, S.U, kStride, kc, kRows, false);
      wait_b();
      tc::fence_async_shared();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after();
        issue_chunk(S, tbase + kColV, false, false, kc == 0);
      }
      mma_round(&mbar, phase);
      __syncthreads();
    }
    // ---- epilogue 1 (warps 0-3, thread = row): v = V + r, reference-order score
    const int m = qrow;
    const float* relr = relsh;
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    bool bad = false;
    if (tid < kEpi) {
      float v[16];
      for (int c = 0; c < dr; c += 16) {
        tc::tmem_ld16(tbase + lane_addr + kColV + c, v);
#pragma unroll
        for (int q = 0; q < 16; q += 4) {
          const float x0 = __fadd_rn(v[q], relr[c + q]), x1 = __fadd_rn(v[q + 1], relr[c + q + 1]);
          const float x2 = __fadd_rn(v[q + 2], relr[c + q + 2]), x3 = __fadd_rn(v[q + 3], relr[c + q + 3]);
          bad |= nonfinite(x0) | nonfinite(x1) | nonfinite(x2) | nonfinite(x3);
          s0 = __fadd_rn(s0, norm_term<L2>(x0));
          s1 = __fadd_rn(s1, norm_term<L2>(x1));
          s2 = __fadd_rn(s2, norm_term<L2>(x2));
          s3 = __fadd_rn(s3, norm_term<L2>(x3));
          if (MODE == kScore && rrow[m] >= 0) {
            float* dst = f.res + static_cast<size_t>(rrow[m]) * dr + c + q;
            dst[0] = x0, dst[1] = x1, dst[2] = x2, dst[3] = x3;
          }
        }
      }
    }
    const float ssum = __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));  // norms.hpp:33 (d >= 8)
    if (tid < kEpi) {
      rs[m] = ssum;
      if (bad && rrow[m] >= 0) pend |= kPendEntity;
    }
    __syncthreads();
    if (tid < kEpi) {
      const int row2 = rrow[m];
      float up = 0.f;
      if (MODE == kTrain) {
        const int kk = m & 63;
        if (kk < np) {
          const float ps = L2 ? __fsqrt_rn(rs[kk]) : rs[kk];
          const float ns = L2 ? __fsqrt_rn(rs[64 + kk]) : rs[64 + kk];
          if (__fsub_rn(__fadd_rn(f.margin, ps), ns) > 0.f) up = m < 64 ? f.unit : -f.unit;
        }
      } else if (row2 >= 0) {
        f.scores[row2] = L2 ? __fsqrt_rn(ssum) : ssum;
        if (MODE == kPrep) up = f.upstream[row2];
      }
      rsc[m] = up == 0.f ? 0.f : (L2 ? __fdiv_rn(up, __fsqrt_rn(__fadd_rn(ssum, kNormEpsF))) : up);
      if (row2 >= 0 && MODE != kScore) f.scal[row2] = up != 0.f ? 1.f : 0.f;
    }
    if (MODE == kTrain && tid == 0) {
      float tl = 0.f;
      for (int kk = 0; kk < np; ++kk) {
        const float ps = L2 ? __fsqrt_rn(rs[kk]) : rs[kk];
        const float ns = L2 ? __fsqrt_rn(rs[64 + kk]) : rs[64 + kk];
        const float term = __fsub_rn(__fadd_rn(f.margin, ps), ns);
        if (term > 0.f) tl = __fadd_rn(tl, term);
      }
      tile_loss_sh = tl;
    }
    __syncthreads();
    if (MODE == kTrain) lsum = __fadd_rn(lsum, tile_loss_sh);
    if (MODE == kScore) {
      const int row2 = tid < kEpi ? rrow[m] : -1;
      if (row2 >= 0)
        for (int c = 0; c < de; c += 4)
          *reinterpret_cast<float4*>(f.res_u + static_cast<size_t>(row2) * de + c) =
              *reinterpret_cast<const float4*>(S.U + m * kStride + c);
      __syncthreads();
      continue;
    }
    if (tid < kEpi) {  // DZ row (norm_direction) into shared memory
      const float sc = rsc[m];
      float v[16];
      for (int c = 0; c < dr; c += 16) {
        tc::tmem_ld16(tbase + lane_addr + kColV + c, v);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float x = __fadd_rn(v[q], relr[c + q]);
          S.DZ[m * kStride + c + q] =
              sc == 0.f ? 0.f : (L2 ? __fmul_rn(x, sc) : (x > 0.f ? sc : (x < 0.f ? -sc : 0.f)));
        }
      }
    }
    __syncthreads();
    {  // sum(dz) per column: two halves of the rows, combined in fixed order
      const int n = tid & (kD - 1), hr = tid >> 7;
      float cs = 0.f;
      for (int mm = hr * 64; mm < hr * 64 + 64; ++mm) cs = __fadd_rn(cs, S.DZ[mm * kStride + n]);
      colsum[hr][n] = cs;
    }
    __syncthreads();
    if (tid < kD) dr_acc = __fadd_rn(dr_acc, __fadd_rn(colsum[0][tid], colsum[1][tid]));
    // ---- GEMM2: dU = DZ M_r (K = dr); B is M_r read MN-major
    for (int kc = 0; kc < dr; kc += kChunk) {
      load_b(r, 1, kc / kChunk);
      stage_kmajor(S.Ahi, S.Alo, S.DZ, kStride, kc, kRows, false);
      wait_b();
      tc::fence_async_shared();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after();
        issue_chunk(S, tbase + kColDU, false, false, kc == 0);
      }
      mma_round(&mbar, phase);
      __syncthreads();
    }
    {  // epilogue 2 (all warps: row qrow, column half): dU rows of active rows
      const int row2 = rrow[qrow];
      const bool act = row2 >= 0 && rsc[qrow] != 0.f;
      float v[16];
      for (int c = half * 64; c < half * 64 + 64; c += 16) {
        tc::tmem_ld16(tbase + lane_addr + kColDU + c, v);
        if (act) {
          float* dst = f.res_u + static_cast<size_t>(row2) * de + c;
#pragma unroll
          for (int q = 0; q < 16; q += 4) *reinterpret_cast<float4*>(dst + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
        }
      }
    }
    // ---- GEMM3: dM += DZ^T U (K = rows); both operands read MN-major
    for (int kc = 0; kc < kRows; kc += kChunk) {
      stage_kmajor_t(S.Ahi, S.Alo, S.DZ, kStride, kc, false);
      stage_kmajor_t(S.Bhi, S.Blo, S.U, kStride, kc, false);
      tc::fence_async_shared();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after();
        issue_chunk(S, tbase + kColDM, false, false, dm_first && kc == 0);
      }
      mma_round(&mbar, phase);
      __syncthreads();
    }
    dm_first = false;
  }
  if (MODE != kScore && cur_k >= 0) flush(cur_k);

  // ---- loss: one partial per CTA (tile order), last CTA finalizes
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, kTmemCols);
  pend = __reduce_or_sync(kFull, pend);
  if (lane == 0 && pend) {
    atomicOr(&f.err[3], pend);
    __threadfence();
  }
  if (MODE != kTrain || !alive) return;
  __shared__ bool last;
  if (tid == 0) {
    f.block_partial[blockIdx.x] = lsum;
    last = ticket_acq_rel(f.counter) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && warp == 0) {
    float acc = 0.f;
    for (int b = lane; b < static_cast<int>(gridDim.x); b += 32) acc = __fadd_rn(acc, f.block_partial[b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_down_sync(kFull, acc, o));
    if (lane == 0) {
      const float loss = __fdiv_rn(acc, static_cast<float>(f.B));
      f.batch_loss[f.batch] = loss;
      if (f.stamp_end) stamp_now(f.stamp_end);
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

// Per relation segment k: sum the (CTA, relation) run partials j + k over the
// CTAs whose tile range meets the relation's tiles (tile order), then SGD.
__global__ void transr_tc_apply_kernel(const uint32_t* __restrict__ tile_total, const uint32_t* __restrict__ seg_tiles,
                                       const uint32_t* __restrict__ tile_seg, const uint32_t* __restrict__ seg_col,
                                       int64_t N, int G, const float* __restrict__ dm_part,
                                       const float* __restrict__ dr_part, float* __restrict__ proj,
                                       float* __restrict__ rel, const float* __restrict__ lr, bool sgd,
                                       const uint32_t* __restrict__ err) {
  if (err[0] != 0) return;
  const uint32_t k = blockIdx.x;
  if (k >= tile_total[1]) return;
  const uint32_t T = tile_total[0];
  const uint32_t lo = seg_tiles[k], hi = seg_tiles[k + 1];
  if (hi <= lo) return;
  const int64_t r = static_cast<int64_t>(seg_col[tile_seg[lo]]) - N;
  const float step = *lr;
  // CTAs whose tile range [T j / G, T (j+1) / G) meets [lo, hi): a contiguous
  // j interval (ranges are monotone); empty ranges own no slot.
  __shared__ unsigned char own[1024];
  __shared__ int jl[1024];
  __shared__ int nj;
  for (int j = threadIdx.x; j < G && j < 1024; j += blockDim.x) {
    const uint32_t a0 = static_cast<uint32_t>((static_cast<uint64_t>(T) * j) / G);
    const uint32_t a1 = static_cast<uint32_t>((static_cast<uint64_t>(T) * (j + 1)) / G);
    own[j] = (a0 < a1 && a1 > lo && a0 < hi) ? 1 : 0;
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // ordered compaction, one warp
    int c = 0;
    for (int j0 = 0; j0 < G && j0 < 1024; j0 += 32) {
      const int j = j0 + static_cast<int>(threadIdx.x);
      const bool o = j < G && j < 1024 && own[j];
      const unsigned m = __ballot_sync(kFull, o);
      if (o) jl[c + __popc(m & lanemask_lt())] = j;
      c += __popc(m);
    }
    if (threadIdx.x == 0) nj = c;
  }
  __syncthreads();
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < kD * kD + kD; i += gridDim.y * blockDim.x) {
    float g = 0.f;
    for (int q = 0; q < nj; ++q) {
      const size_t slot = static_cast<size_t>(jl[q]) + k;
      g = __fadd_rn(g, i < kD * kD ? dm_part[slot * kD * kD + i] : dr_part[slot * kD + (i - kD * kD)]);
    }
    float* p = i < kD * kD ? proj + r * kD * kD + i : rel + r * kD + (i - kD * kD);
    *p = sgd ? __fsub_rn(*p, __fmul_rn(step, g)) : __fadd_rn(*p, g);
  }
}

// ---- self-test GEMM: D[m][n] = sum_k A(m,k) B(n,k) through each operand view
// mode 0: A [m][k], B [n][k] (both K-major)    -> GEMM1 shape
// mode 1: A [m][k], B [k][n] (B MN-major)      -> GEMM2 shape
// mode 2: A [k][m], B [k][n] (both MN-major)   -> GEMM3 shape
__global__ void __launch_bounds__(kThreads, 1) tc_selftest_kernel(int mode, const float* A, const float* B, float* D) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc::tmem_alloc(&tmem_base, kTmemCols);
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    tc::fence_barrier_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  uint32_t phase = 0;
  for (int kc = 0; kc < kD; kc += kChunk) {
    if (mode == 2) stage_kmajor_t(S.Ahi, S.Alo, A, kD, kc, true);
    else stage_kmajor(S.Ahi, S.Alo, A, kD, kc, kRows, true);
    if (mode == 0) stage_kmajor(S.Bhi, S.Blo, B, kD, kc, kD, true);
    else stage_kmajor_t(S.Bhi, S.Blo, B, kD, kc, true);
    tc::fence_async_shared();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
      issue_chunk(S, tmem_base, false, false, kc == 0);
    }
    mma_round(&mbar, phase);
    __syncthreads();
  }
  float v[16];
  if (warp < 4)
    for (int c = 0; c < kD; c += 16) {
      tc::tmem_ld16(tmem_base + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
      for (int q = 0; q < 16; ++q) D[tid * kD + c + q] = v[q];
    }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem_base, kTmemCols);
}

template <bool L2, int MODE>
void configure_one() {
  SKG_CUDA(cudaFuncSetAttribute(transr_tc_kernel<L2, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(Smem))));
}

}  // namespace

bool transr_tc_supported(int de, int dr) { return de == kD && dr == kD; }

void configure_transr_tc_kernels() {
  configure_one<true, kTrain>();
  configure_one<true, kScore>();
  configure_one<true, kPrep>();
  configure_one<false, kTrain>();
  configure_one<false, kScore>();
  configure_one<false, kPrep>();
  SKG_CUDA(cudaFuncSetAttribute(tc_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(Smem))));
}

int64_t transr_tc_slots(int num_sms, int64_t R) { return num_sms + R + 2; }

int64_t transr_tc_mr_floats(int64_t R) { return R * kMrFloatsPerRel; }

void launch_transr_tc(bool l2, int mode, const FwdArgs& fa, const uint32_t* ent_val, const uint32_t* seg_start,
                      const uint32_t* seg_col, const uint32_t* tile_seg, const uint32_t* tile_p0,
                      const uint32_t* tile_total, const uint32_t* seg_tiles, float* dm_part, float* dr_part,
                      float* mr_chunks, int64_t R, int num_sms, cudaStream_t s) {
  transr_prep_mr_kernel<<<dim3(static_cast<unsigned>(R), 8), 256, 0, s>>>(fa.proj, mr_chunks);
  count_launch();
  TcArgs a{};
  a.mr_chunks = mr_chunks;
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
  const size_t smem = sizeof(Smem);
  if (l2) {
    if (mode == kTrain) transr_tc_kernel<true, kTrain><<<num_sms, kThreads, smem, s>>>(a);
    else if (mode == kScore) transr_tc_kernel<true, kScore><<<num_sms, kThreads, smem, s>>>(a);
    else transr_tc_kernel<true, kPrep><<<num_sms, kThreads, smem, s>>>(a);
  } else {
    if (mode == kTrain) transr_tc_kernel<false, kTrain><<<num_sms, kThreads, smem, s>>>(a);
    else if (mode == kScore) transr_tc_kernel<false, kScore><<<num_sms, kThreads, smem, s>>>(a);
    else transr_tc_kernel<false, kPrep><<<num_sms, kThreads, smem, s>>>(a);
  }
  count_launch();
  SKG_LAUNCH_CHECK();
}

void launch_transr_tc_apply(const uint32_t* tile_total, const uint32_t* seg_tiles, const uint32_t* tile_seg,
                            const uint32_t* seg_col, int64_t N, int G, const float* dm_part, const float* dr_part,
                            float* proj, float* rel, const float* lr, bool sgd, const uint32_t* err, int64_t R,
                            cudaStream_t s) {
  transr_tc_apply_kernel<<<dim3(static_cast<unsigned>(R), 16), 256, 0, s>>>(tile_total, seg_tiles, tile_seg, seg_col, N,
                                                                           G, dm_part, dr_part, proj, rel, lr, sgd, err);
  count_launch();
  SKG_LAUNCH_CHECK();
}

void transr_tc_selftest(int mode, const float* A, const float* B, float* D, cudaStream_t s) {
  tc_selftest_kernel<<<1, kThreads, sizeof(Smem), s>>>(mode, A, B, D);
  count_launch();
  SKG_LAUNCH_CHECK();
}

}  // namespace skg
