// Epoch plan construction (see plan.cuh).
#include "common.cuh"
#include "plan.cuh"

namespace skg {

namespace {

__device__ __forceinline__ uint32_t col_key(int64_t col, int64_t N, int64_t Rn) {
  // relation columns first: long segments start early in the backward grid
  return static_cast<uint32_t>(col >= N ? col - N : col + Rn);
}

// Entries that do not exist (the cancelled entity pair of a self-loop row, the
// relation entry of an ht-layout row) get the per-batch dummy column N + Rn:
// it sorts after every real column of its batch, forms one segment with
// seg_col = kDummyCol that every consumer skips, and keeps all batches'
// entries inside their own block-aligned range (segmented radix sort).
__device__ __forceinline__ void emit_row(uint32_t* key, uint32_t* val, int64_t base, uint32_t bkey,
                                         int32_t h, int32_t t, int32_t r, uint32_t row2, int64_t N,
                                         int64_t Rn, bool with_rel) {
  const uint32_t dummy = bkey | static_cast<uint32_t>(N + Rn);
  if (h != t) {  // +1 and -1 cancel at coo_to_csr time (sparse.hpp:145-155)
    key[base] = bkey | col_key(h, N, Rn);
    val[base] = row2;
    key[base + 1] = bkey | col_key(t, N, Rn);
    val[base + 1] = row2 | 0x80000000u;
  } else {
    key[base] = dummy;
    val[base] = 0;
    key[base + 1] = dummy;
    val[base + 1] = 0;
  }
  key[base + 2] = with_rel ? (bkey | col_key(N + r, N, Rn)) : dummy;
  val[base + 2] = row2;
}

// One thread per epoch position k: the triple's packed ids {h, t, nh, nt}
// (one 16-byte read instead of four scattered 4-byte ones) and its relation
// give the pair record and the positive and negative rows' entries.
__global__ void gen_train_entries_kernel(const int32_t* __restrict__ order, const int4* __restrict__ quad,
                                         const int32_t* __restrict__ R, int64_t M, int64_t B, int64_t N,
                                         int64_t Rn, int cb, uint32_t* __restrict__ key,
                                         uint32_t* __restrict__ val, int4* __restrict__ pair_ht,
                                         int32_t* __restrict__ pair_r) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < M;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = k / B, i = k - b * B;
    const int64_t Bb = min(B, M - b * B);
    const int32_t id = __ldg(order + k);
    const int4 q = __ldg(quad + id);
    const int32_t r = __ldg(R + id);
    pair_ht[k] = q;
    pair_r[k] = r;
    const uint32_t bkey = static_cast<uint32_t>(b) << cb;
    emit_row(key, val, 6 * b * B + 3 * i, bkey, q.x, q.y, r, static_cast<uint32_t>(i), N, Rn, true);
    emit_row(key, val, 6 * b * B + 3 * (Bb + i), bkey, q.z, q.w, r, static_cast<uint32_t>(Bb + i), N, Rn, true);
  }
}

__global__ void pack_quad_kernel(const int32_t* __restrict__ H, const int32_t* __restrict__ T,
                                 const int32_t* __restrict__ NH, const int32_t* __restrict__ NT, int64_t M,
                                 int4* __restrict__ quad) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < M;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    quad[i] = make_int4(H[i], T[i], NH[i], NT[i]);
}

__global__ void gen_batch_entries_kernel(const int32_t* __restrict__ H, const int32_t* __restrict__ R,
                                         const int32_t* __restrict__ T, int64_t m, int64_t N,
                                         int64_t Rn, bool with_rel,
                                         uint32_t* __restrict__ key, uint32_t* __restrict__ val) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    emit_row(key, val, 3 * i, 0u, H[i], T[i], R[i], static_cast<uint32_t>(i), N, Rn, with_rel);
}

__global__ void seg_flag_kernel(const uint32_t* __restrict__ key, int64_t E, uint32_t invalid,
                                uint32_t* __restrict__ flag) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < E;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t k = key[e];
    flag[e] = (k != invalid && (e == 0 || key[e - 1] != k)) ? 1u : 0u;
  }
}

__global__ void seg_fill_kernel(const uint32_t* __restrict__ key, const uint32_t* __restrict__ flag,
                                const uint32_t* __restrict__ segid, int64_t E, uint32_t invalid,
                                int cb, int64_t N, int64_t Rn, int64_t nb,
                                const uint32_t* __restrict__ nseg, uint32_t* __restrict__ seg_start,
                                uint32_t* __restrict__ seg_col, uint32_t* __restrict__ seg_base) {
  const uint32_t cmask = (1u << cb) - 1u;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < E;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t k = key[e];
    if (k == invalid) continue;
    if (flag[e]) {
      const uint32_t sidx = segid[e];
      seg_start[sidx] = static_cast<uint32_t>(e);
      const int64_t cp = k & cmask;
      seg_col[sidx] = cp == N + Rn ? kDummyCol : static_cast<uint32_t>(cp < Rn ? N + cp : cp - Rn);
      const uint32_t b = k >> cb;
      if (e == 0 || (key[e - 1] >> cb) != b) seg_base[b] = sidx;
    }
    if (e + 1 == E || key[e + 1] == invalid) {
      seg_start[*nseg] = static_cast<uint32_t>(e + 1);
      seg_base[nb] = *nseg;
    }
  }
}

int grid_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return static_cast<int>(b < 1 ? 1 : (b > 8192 ? 8192 : b));
}

// seg_items: entries per batch when every batch starts on a sort block
// boundary (the sort then orders columns inside each batch only), else 0.
void finish_plan(EpochPlan& p, int64_t seg_items, int64_t N, int64_t Rn, cudaStream_t s) {
  const uint32_t invalid = 0xFFFFFFFFu;  // never a key (keys use <= 31 bits)
  const bool seg = seg_items > 0 && p.nb > 1 && radix_segment_ok(seg_items, p.E);
  const bool alt = radix_sort_pairs(p.key, p.val, p.key_alt, p.val_alt, p.E, seg ? p.cb : p.kb + p.cb, p.sort, s,
                                    seg ? seg_items : 0);
  const uint32_t* k = alt ? p.key_alt : p.key;
  p.sorted_val = alt ? p.val_alt : p.val;
  // the unsorted pair of buffers is free now: flags and segment ids live there
  uint32_t* flag = alt ? p.key : p.key_alt;
  uint32_t* segid = alt ? p.val : p.val_alt;
  seg_flag_kernel<<<grid_for(p.E), 256, 0, s>>>(k, p.E, invalid, flag);
  count_launch();
  SKG_LAUNCH_CHECK();
  exclusive_scan_u32(flag, segid, p.E, p.nseg, p.scan, s);
  SKG_CUDA(cudaMemsetAsync(p.seg_base, 0, sizeof(uint32_t) * (p.nb + 1), s));
  seg_fill_kernel<<<grid_for(p.E), 256, 0, s>>>(k, flag, segid, p.E, invalid, p.cb, N, Rn, p.nb, p.nseg,
                                                p.seg_start, p.seg_col, p.seg_base);
  count_launch();
  SKG_LAUNCH_CHECK();
}

}  // namespace

void EpochPlan::reserve(int64_t entries, int64_t batches) {
  if (entries > cap_entries) {
    for (uint32_t** b : {&key, &val, &key_alt, &val_alt, &seg_start, &seg_col}) {
      if (*b) cudaFree(*b);
      SKG_CUDA(cudaMalloc(b, sizeof(uint32_t) * (entries + 1)));
    }
    if (!nseg) SKG_CUDA(cudaMalloc(&nseg, sizeof(uint32_t)));
    sort.reserve(entries);
    scan.reserve(entries);
    cap_entries = entries;
  }
  if (entries / 6 + 1 > cap_pairs) {
    if (pair_ht) cudaFree(pair_ht);
    if (pair_r) cudaFree(pair_r);
    cap_pairs = entries / 6 + 1;
    SKG_CUDA(cudaMalloc(&pair_ht, sizeof(int4) * cap_pairs));
    SKG_CUDA(cudaMalloc(&pair_r, sizeof(int32_t) * cap_pairs));
  }
  if (batches > cap_batches) {
    if (seg_base) cudaFree(seg_base);
    SKG_CUDA(cudaMalloc(&seg_base, sizeof(uint32_t) * (batches + 1)));
    cap_batches = batches;
  }
}

void EpochPlan::release() {
  for (uint32_t** b : {&key, &val, &key_alt, &val_alt, &seg_start, &seg_col, &seg_base, &nseg}) {
    if (*b) cudaFree(*b);
    *b = nullptr;
  }
  if (pair_ht) cudaFree(pair_ht);
  if (pair_r) cudaFree(pair_r);
  pair_ht = nullptr;
  pair_r = nullptr;
  cap_entries = cap_batches = cap_pairs = 0;
  sort.release();
  scan.release();
}

void pack_triple_quads(const int32_t* H, const int32_t* T, const int32_t* NH, const int32_t* NT, int64_t M,
                       int4* quad, cudaStream_t s) {
  if (M <= 0) return;
  pack_quad_kernel<<<grid_for(M), 256, 0, s>>>(H, T, NH, NT, M, quad);
  count_launch();
  SKG_LAUNCH_CHECK();
}

void build_epoch_plan(const int32_t* order, const int4* quad, const int32_t* R, int64_t M, int64_t B, int64_t N,
                      int64_t Rn, EpochPlan& p, cudaStream_t s) {
  p.nb = (M + B - 1) / B;
  p.E = 6 * M;
  p.kb = bits_for(static_cast<uint64_t>(p.nb - 1));
  p.cb = bits_for(static_cast<uint64_t>(N + Rn));  // + the dummy column N + Rn
  if (p.kb + p.cb > 31) throw CudaError("epoch plan: batches x columns exceed the 31-bit key space");
  p.reserve(p.E, p.nb);
  gen_train_entries_kernel<<<grid_for(M), 256, 0, s>>>(order, quad, R, M, B, N, Rn, p.cb, p.key, p.val, p.pair_ht,
                                                       p.pair_r);
  count_launch();
  SKG_LAUNCH_CHECK();
  finish_plan(p, 6 * B, N, Rn, s);
}

void build_batch_plan(const int32_t* H, const int32_t* R, const int32_t* T, int64_t m, int64_t N,
                      int64_t Rn, int layout, EpochPlan& p, cudaStream_t s) {
  p.nb = 1;
  p.E = 3 * m;
  p.kb = 0;
  p.cb = bits_for(static_cast<uint64_t>(N + Rn));
  p.reserve(p.E, 1);
  gen_batch_entries_kernel<<<grid_for(m), 256, 0, s>>>(H, R, T, m, N, Rn, layout == 1, p.key, p.val);
  count_launch();
  SKG_LAUNCH_CHECK();
  finish_plan(p, 0, N, Rn, s);
}

}  // namespace skg
