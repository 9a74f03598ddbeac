// The reference's generic plus-times sparse operators on device, for callers
// of the reference API that use them directly (sparse.hpp:110-306):
// coo_to_csr, transpose, spmm and spmm_transpose_add. The training path never
// calls these (its incidence plan is built in plan.cu); they keep the C ABI a
// drop-in for the whole sparse layer the trainer is built from.
//
// Ordering contracts that make them bit-exact with the reference:
//  - coo_to_csr (sparse.hpp:110-161): entries are bucketed by row in input
//    order (the reference's cursor scatter), then each row is ordered by column
//    and duplicates are summed left to right and dropped when they cancel to
//    exactly zero. The per-row order is a stable insertion sort, which is what
//    libstdc++'s std::sort does for rows of at most 16 entries (its final
//    insertion-sort pass; introsort partitioning only starts above 16), so the
//    summation order of duplicates matches for every such row (incidence rows
//    hold at most 3 entries).
//  - transpose (sparse.hpp:164-183): a stable counting sort over columns, so
//    each transposed row lists its source rows ascending.
//  - spmm (sparse.hpp:211-266): one warp per output row; the 0/1/2/3-entry
//    cases are the reference's fused expressions (left-to-right), longer rows
//    accumulate from zero in stored order. No FMA contraction.
//  - spmm_transpose_add (sparse.hpp:273-306): one warp per column of A, the
//    sink row accumulates a * g_row over ascending source rows.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"
#include "primitives.cuh"

namespace skg {

namespace {

int grid_n(int64_t n, int per_block = 256) {
  const int64_t b = (n + per_block - 1) / per_block;
  return static_cast<int>(b < 1 ? 1 : (b > 8192 ? 8192 : b));
}

template <class T>
struct Tmp {  // scoped device scratch
  T* p = nullptr;
  explicit Tmp(int64_t n) { SKG_CUDA(cudaMalloc(&p, sizeof(T) * (n > 0 ? n : 1))); }
  ~Tmp() {
    if (p) cudaFree(p);
  }
  Tmp(const Tmp&) = delete;
  Tmp& operator=(const Tmp&) = delete;
};

__global__ void iota_keyed_kernel(const int64_t* __restrict__ key_src, int64_t n, uint32_t* __restrict__ key,
                                  uint32_t* __restrict__ val) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    key[i] = static_cast<uint32_t>(key_src[i]);
    val[i] = static_cast<uint32_t>(i);
  }
}

// counts[k] = #{i : key_src[i] == k} (integer atomics: order-free, exact)
__global__ void histogram_kernel(const int64_t* __restrict__ key_src, int64_t n, uint32_t* __restrict__ counts) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicAdd(counts + key_src[i], 1u);
}

// Per row: gather the row's entries (input order), stable insertion sort by
// column, merge duplicates left to right, drop exact zeros; the merged row is
// left at the start of the row's bucket and its length in merged[r].
__global__ void coo_rows_kernel(const uint32_t* __restrict__ order, const uint32_t* __restrict__ start,
                                const int64_t* __restrict__ cols, const float* __restrict__ vals, int64_t rows,
                                int64_t* __restrict__ bcol, float* __restrict__ bval, uint32_t* __restrict__ merged) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t lo = start[r], hi = start[r + 1];
    for (int64_t p = lo; p < hi; ++p) {  // insertion sort, stable (strict < moves left)
      const uint32_t i = order[p];
      const int64_t c = cols[i];
      const float v = vals[i];
      int64_t q = p;
      while (q > lo && c < bcol[q - 1]) {
        bcol[q] = bcol[q - 1];
        bval[q] = bval[q - 1];
        --q;
      }
      bcol[q] = c;
      bval[q] = v;
    }
    int64_t w = lo;
    for (int64_t p = lo; p < hi;) {
      const int64_t c = bcol[p];
      float v = bval[p++];
      while (p < hi && bcol[p] == c) v = __fadd_rn(v, bval[p++]);
      if (v != 0.f) {
        bcol[w] = c;
        bval[w] = v;
        ++w;
      }
    }
    merged[r] = static_cast<uint32_t>(w - lo);
  }
}

__global__ void coo_emit_kernel(const uint32_t* __restrict__ start, const uint32_t* __restrict__ merged,
                                const uint32_t* __restrict__ out_off, const int64_t* __restrict__ bcol,
                                const float* __restrict__ bval, int64_t rows, int64_t* __restrict__ row_ptr,
                                int64_t* __restrict__ col, float* __restrict__ val, const uint32_t* __restrict__ total) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t o = out_off[r], lo = start[r];
    row_ptr[r] = o;
    for (uint32_t k = 0; k < merged[r]; ++k) {
      col[o + k] = bcol[lo + k];
      val[o + k] = bval[lo + k];
    }
    if (r == rows - 1) row_ptr[rows] = *total;
  }
}

// source row of every CSR entry
__global__ void expand_rows_kernel(const int64_t* __restrict__ row_ptr, int64_t rows, uint32_t* __restrict__ row_of) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    for (int64_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) row_of[p] = static_cast<uint32_t>(r);
}

__global__ void transpose_emit_kernel(const uint32_t* __restrict__ sorted_p, const uint32_t* __restrict__ row_of,
                                      const float* __restrict__ vals, int64_t nnz, int64_t* __restrict__ tcol,
                                      float* __restrict__ tval) {
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < nnz;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t p = sorted_p[q];
    tcol[q] = row_of[p];
    tval[q] = vals[p];
  }
}

__global__ void widen_scan_kernel(const uint32_t* __restrict__ off, int64_t n, const uint32_t* __restrict__ total,
                                  int64_t* __restrict__ row_ptr) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i <= n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    row_ptr[i] = i < n ? off[i] : *total;
}

// warp per output row; lanes stride the d coordinates
__global__ void spmm_kernel(const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ col,
                            const float* __restrict__ a, int64_t rows, int d, const float* __restrict__ x,
                            float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; i < rows;
       i += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t b = row_ptr[i], e = row_ptr[i + 1];
    float* o = out + i * d;
    for (int j = lane; j < d; j += 32) {
      float v;
      switch (e - b) {
        case 0: v = 0.f; break;
        case 1: v = __fmul_rn(a[b], x[col[b] * d + j]); break;
        case 2:
          v = __fadd_rn(__fmul_rn(a[b], x[col[b] * d + j]), __fmul_rn(a[b + 1], x[col[b + 1] * d + j]));
          break;
        case 3:
          v = __fadd_rn(__fadd_rn(__fmul_rn(a[b], x[col[b] * d + j]), __fmul_rn(a[b + 1], x[col[b + 1] * d + j])),
                        __fmul_rn(a[b + 2], x[col[b + 2] * d + j]));
          break;
        default:
          v = 0.f;
          for (int64_t p = b; p < e; ++p) v = __fadd_rn(v, __fmul_rn(a[p], x[col[p] * d + j]));
          break;
      }
      o[j] = v;
    }
  }
}

// warp per column k of A (row of A^T): sink_k += sum over ascending source rows
__global__ void spmm_t_add_kernel(const int64_t* __restrict__ trow_ptr, const int64_t* __restrict__ tcol,
                                  const float* __restrict__ ta, int64_t cols, int d, const float* __restrict__ g,
                                  float* __restrict__ sink) {
  const int lane = threadIdx.x & 31;
  for (int64_t k = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; k < cols;
       k += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t b = trow_ptr[k], e = trow_ptr[k + 1];
    if (b == e) continue;
    float* o = sink + k * d;
    for (int j = lane; j < d; j += 32) {
      float v = o[j];
      for (int64_t p = b; p < e; ++p) v = __fadd_rn(v, __fmul_rn(ta[p], g[tcol[p] * d + j]));
      o[j] = v;
    }
  }
}

// Stable counting sort of entries by a u32 key < 2^bits: returns the entry
// order (indices into the input) in `order` (n entries, device).
void stable_order_by(const int64_t* key_src, int64_t n, int bits, uint32_t* order, cudaStream_t s) {
  Tmp<uint32_t> k(n), v(n), k2(n), v2(n);
  iota_keyed_kernel<<<grid_n(n), 256, 0, s>>>(key_src, n, k.p, v.p);
  count_launch();
  SKG_LAUNCH_CHECK();
  SortPlan sp;
  sp.reserve(n);
  const bool alt = radix_sort_pairs(k.p, v.p, k2.p, v2.p, n, std::max(1, bits), sp, s);
  SKG_CUDA(cudaMemcpyAsync(order, alt ? v2.p : v.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s));
  SKG_CUDA(cudaStreamSynchronize(s));  // scratch is freed on return
}

// Exclusive offsets of a per-key histogram: off[k] (n_keys + 1 entries incl. total).
void key_offsets(const int64_t* key_src, int64_t n, int64_t n_keys, uint32_t* off, uint32_t* total, cudaStream_t s) {
  Tmp<uint32_t> cnt(n_keys + 1);
  SKG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(uint32_t) * (n_keys + 1), s));
  if (n > 0) {
    histogram_kernel<<<grid_n(n), 256, 0, s>>>(key_src, n, cnt.p);
    count_launch();
    SKG_LAUNCH_CHECK();
  }
  ScanPlan sc;
  sc.reserve(n_keys + 1);
  exclusive_scan_u32(cnt.p, off, n_keys + 1, total, sc, s);
  SKG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

void sparse_coo_to_csr(int64_t rows, int64_t cols, int64_t nnz, const int64_t* d_rows, const int64_t* d_cols,
                       const float* d_vals, int64_t* d_row_ptr, int64_t* d_col, float* d_val, int64_t* nnz_out,
                       cudaStream_t s) {
  (void)cols;
  Tmp<uint32_t> order(nnz), start(rows + 1), merged(rows + 1), out_off(rows + 1), tot(2);
  Tmp<int64_t> bcol(nnz);
  Tmp<float> bval(nnz);
  if (nnz > 0) stable_order_by(d_rows, nnz, bits_for(static_cast<uint64_t>(rows)), order.p, s);
  key_offsets(d_rows, nnz, rows, start.p, tot.p, s);
  if (rows > 0) {
    coo_rows_kernel<<<grid_n(rows, 128), 128, 0, s>>>(order.p, start.p, d_cols, d_vals, rows, bcol.p, bval.p,
                                                      merged.p);
    count_launch();
    SKG_LAUNCH_CHECK();
    ScanPlan sc;
    sc.reserve(rows);
    exclusive_scan_u32(merged.p, out_off.p, rows, tot.p + 1, sc, s);
    coo_emit_kernel<<<grid_n(rows), 256, 0, s>>>(start.p, merged.p, out_off.p, bcol.p, bval.p, rows, d_row_ptr, d_col,
                                                 d_val, tot.p + 1);
    count_launch();
    SKG_LAUNCH_CHECK();
    uint32_t z = 0;
    SKG_CUDA(cudaMemcpyAsync(&z, tot.p + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    SKG_CUDA(cudaStreamSynchronize(s));
    *nnz_out = z;
  } else {
    SKG_CUDA(cudaMemsetAsync(d_row_ptr, 0, sizeof(int64_t), s));
    SKG_CUDA(cudaStreamSynchronize(s));
    *nnz_out = 0;
  }
}

void sparse_transpose(int64_t rows, int64_t cols, int64_t nnz, const int64_t* d_row_ptr, const int64_t* d_col,
                      const float* d_val, int64_t* d_trow_ptr, int64_t* d_tcol, float* d_tval, cudaStream_t s) {
  Tmp<uint32_t> off(cols + 1), tot(1), order(nnz), row_of(nnz);
  key_offsets(d_col, nnz, cols, off.p, tot.p, s);
  widen_scan_kernel<<<grid_n(cols + 1), 256, 0, s>>>(off.p, cols, tot.p, d_trow_ptr);
  count_launch();
  SKG_LAUNCH_CHECK();
  if (nnz > 0) {
    stable_order_by(d_col, nnz, bits_for(static_cast<uint64_t>(cols)), order.p, s);
    expand_rows_kernel<<<grid_n(rows), 256, 0, s>>>(d_row_ptr, rows, row_of.p);
    transpose_emit_kernel<<<grid_n(nnz), 256, 0, s>>>(order.p, row_of.p, d_val, nnz, d_tcol, d_tval);
    count_launch(2);
    SKG_LAUNCH_CHECK();
  }
  SKG_CUDA(cudaStreamSynchronize(s));
}

void sparse_spmm(int64_t rows, const int64_t* d_row_ptr, const int64_t* d_col, const float* d_val, int d,
                 const float* d_x, float* d_out, int num_sms, cudaStream_t s) {
  if (rows <= 0 || d <= 0) return;
  const int blocks = static_cast<int>(std::min<int64_t>((rows * 32 + 255) / 256, 16LL * num_sms));
  spmm_kernel<<<blocks, 256, 0, s>>>(d_row_ptr, d_col, d_val, rows, d, d_x, d_out);
  count_launch();
  SKG_LAUNCH_CHECK();
}

void sparse_spmm_transpose_add(int64_t rows, int64_t cols, int64_t nnz, const int64_t* d_row_ptr,
                               const int64_t* d_col, const float* d_val, int d, const float* d_g, float* d_sink,
                               int num_sms, cudaStream_t s) {
  if (cols <= 0 || d <= 0 || nnz <= 0) return;
  Tmp<int64_t> trp(cols + 1), tcol(nnz);
  Tmp<float> tval(nnz);
  sparse_transpose(rows, cols, nnz, d_row_ptr, d_col, d_val, trp.p, tcol.p, tval.p, s);
  const int blocks = static_cast<int>(std::min<int64_t>((cols * 32 + 255) / 256, 16LL * num_sms));
  spmm_t_add_kernel<<<blocks, 256, 0, s>>>(trp.p, tcol.p, tval.p, cols, d, d_g, d_sink);
  count_launch();
  SKG_LAUNCH_CHECK();
  SKG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace skg
