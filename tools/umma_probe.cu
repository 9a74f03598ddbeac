// Standalone tcgen05 kind::tf32 probe (sm_100a): operand-view correctness of
// one physical no-swizzle layout read K-major and MN-major, fp32->tf32
// operand conversion (truncate vs round), and MMA issue throughput vs N.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe tools/umma_probe.cu && ./umma_probe
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t mdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int amn, int bmn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amn << 15) | ((uint32_t)bmn << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
               ::"r"(d), "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ss_el(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* m) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(m)) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(m)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t ph) {
  asm volatile("{\n\t.reg .pred d;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n\t@!d bra W_%=;\n\t}\n" ::"r"(su32(m)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t n) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(dst)), "r"(n) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t b, uint32_t n) { asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(b), "r"(n) : "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
                 "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               ::"r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])),
                 "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
                 "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
                 "r"(__float_as_uint(v[15])) : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Physical layout P(a, c) of a 128 x 128 fp32 tile: 16-byte unit (a%8) + (a/8)*R8 + (c/4)*C4, element c%4.
constexpr int R8 = 256, C4 = 8;  // units
__host__ __device__ inline int poff(int a, int c) { return (((a & 7) + (a >> 3) * R8 + (c >> 2) * C4) << 2) + (c & 3); }
// K-major view (row = a, k = c): LBO = C4, SBO = R8.  MN-major view (mn = c, k = a): LBO = R8, SBO = C4.
constexpr uint32_t KM_LBO = C4 * 16, KM_SBO = R8 * 16;
__device__ uint32_t MN_LBO = R8 * 16, MN_SBO = C4 * 16;

// D[m][n] = sum_k A(m,k) B(n,k). A stored as P(m,k) (amn=0) or P(k,m) (amn=1); B as P(n,k) or P(k,n).
// ts=1: A from TMEM (lane m, column k) instead of smem.
__global__ void gemm_probe(const float* A, const float* B, float* D, int amn, int bmn, int ts) {
  extern __shared__ __align__(1024) float sm[];
  float* sA = sm;
  float* sB = sm + 128 * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 128; i += blockDim.x) {
    const int r = i / 128, c = i % 128;  // A[r][c] logical: r = m, c = k
    sA[amn ? poff(c, r) : poff(r, c)] = A[i];
    sB[bmn ? poff(c, r) : poff(r, c)] = B[i];  // B[r][c]: r = n, c = k
  }
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tbase;
  if (ts && warp < 4) {  // A into TMEM columns 256.. (lane = m, column = k)
    float v[16];
    for (int c = 0; c < 128; c += 16) {
      for (int q = 0; q < 16; ++q) v[q] = A[(warp * 32 + (tid & 31)) * 128 + c + q];
      tmem_st16(tb + ((uint32_t)(warp * 32) << 16) + 256 + c, v);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint32_t id = idesc_tf32(128, 128, ts ? 0 : amn, bmn);
    for (int ks = 0; ks < 16; ++ks) {  // K = 8 per MMA
      const uint32_t aoff = amn ? (uint32_t)(ks * 8 / 8) * (R8 * 16) : (uint32_t)(ks * 2) * (C4 * 16);
      const uint32_t boff = bmn ? (uint32_t)(ks) * (R8 * 16) : (uint32_t)(ks * 2) * (C4 * 16);
      const uint64_t bd = mdesc(su32(sB) + boff, bmn ? MN_LBO : KM_LBO, bmn ? MN_SBO : KM_SBO);
      if (ts) mma_ts(tb, tb + 256 + ks * 8, bd, id, ks > 0);
      else mma_ss(tb, mdesc(su32(sA) + aoff, amn ? MN_LBO : KM_LBO, amn ? MN_SBO : KM_SBO), bd, id, ks > 0);
    }
    commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    float v[16];
    for (int c = 0; c < 128; c += 16) {
      tmem_ld16(tb + ((uint32_t)(warp * 32) << 16) + c, v);
      for (int q = 0; q < 16; ++q) D[(warp * 32 + (tid & 31)) * 128 + c + q] = v[q];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}

__global__ void rate_warp(int N, int iters, long long* cyc) {
  extern __shared__ __align__(1024) float sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 3 * 128 * 128; i += blockDim.x) sm[i] = 0.f;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tbase;
  if (warp == 0) {
    const uint32_t id = idesc_tf32(128, N, 0, 0);
    const uint32_t sa = su32(sm), sb = su32(sm + 128 * 128);
    const uint64_t a0 = mdesc(sa, KM_LBO, KM_SBO), b0 = mdesc(sb, KM_LBO, KM_SBO);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) {
        const uint64_t step = (uint64_t)((ks * 2 * C4 * 16) >> 4);
        mma_ss_el(tb, a0 + step, b0 + step, id, 1);
      }
    }
    if (tid == 0) commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (tid == 0) cyc[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}

// Throughput: iters x 16 MMAs (K = 8 each) of M=128 x N, smem operands (or A in TMEM).
__global__ void rate_probe(int N, int iters, int amn, int bmn, int ts, long long* cyc, int ndst) {
  extern __shared__ __align__(1024) float sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 3 * 128 * 128; i += blockDim.x) sm[i] = 0.f;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tbase;
  if (tid == 0) {
    const uint32_t id = idesc_tf32(128, N, ts ? 0 : amn, bmn);
    const uint32_t sa = su32(sm), sb = su32(sm + 128 * 128);
    uint64_t ad[16], bd[16];
#pragma unroll
    for (int ks = 0; ks < 16; ++ks) {
      const uint32_t aoff = amn ? ks * (R8 * 16) : ks * 2 * (C4 * 16);
      const uint32_t boff = bmn ? ks * (R8 * 16) : ks * 2 * (C4 * 16);
      bd[ks] = mdesc(sb + boff, bmn ? MN_LBO : KM_LBO, bmn ? MN_SBO : KM_SBO);
      ad[ks] = mdesc(sa + aoff, amn ? MN_LBO : KM_LBO, amn ? MN_SBO : KM_SBO);
    }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) {
        if (ts) mma_ts(tb + (it & 1) * 0, tb + 256 + ks * 8, bd[ks], id, 1);
        else mma_ss(tb + (uint32_t)((ks % ndst) * N), ad[ks], bd[ks], id, 1);
      }
    }
    commit(&bar);
    mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}

static float tf32_trunc(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; }
static float tf32_rna(float x) { uint32_t u; memcpy(&u, &x, 4); u += 0x1000u; u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; }

__global__ void decode_probe(const float* A, const float* Bphys, float* D, uint32_t lbo, uint32_t sbo, int nphys) {
  extern __shared__ __align__(1024) float sm[];
  float* sA = sm;
  float* sB = sm + 128 * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 128; i += blockDim.x) sA[poff(i / 128, i % 128)] = A[i];
  for (int i = tid; i < nphys; i += blockDim.x) sB[i] = Bphys[i];
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tbase;
  if (tid == 0) {
    const uint32_t id = idesc_tf32(128, 128, 0, 1);
    // only k-group 0 (k = 0..7): one MMA
    mma_ss(tb, mdesc(su32(sA), KM_LBO, KM_SBO), mdesc(su32(sB), lbo, sbo), id, 0);
    commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    float v[16];
    for (int c = 0; c < 128; c += 16) {
      tmem_ld16(tb + ((uint32_t)(warp * 32) << 16) + c, v);
      for (int q = 0; q < 16; ++q) D[(warp * 32 + (tid & 31)) * 128 + c + q] = v[q];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}

#ifdef DECODE
int main() {
  const size_t smem = 3 * 128 * 128 * 4;
  CK(cudaFuncSetAttribute(decode_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  std::vector<float> A(128 * 128, 0.f), P(2 * 128 * 128), D(128 * 128), D2(128 * 128);
  for (int m = 0; m < 128; ++m) A[m * 128 + m] = 1.f;  // identity: D[m][n] = B(n, k=m) for m < 8
  float *dA, *dP, *dD;
  CK(cudaMalloc(&dA, 65536)); CK(cudaMalloc(&dP, 131072)); CK(cudaMalloc(&dD, 65536));
  CK(cudaMemcpy(dA, A.data(), 65536, cudaMemcpyHostToDevice));
  const uint32_t combos[][2] = {{4096, 128}, {128, 4096}, {128, 128}, {4096, 4096}, {256, 128}, {128, 256}, {1024, 128}, {128, 1024}};
  for (auto& cb : combos) {
    for (int pass = 0; pass < 2; ++pass) {
      for (int i = 0; i < 2 * 128 * 128; ++i) P[i] = pass ? (float)(i / 1024) : (float)(i % 1024);
      CK(cudaMemcpy(dP, P.data(), 131072, cudaMemcpyHostToDevice));
      decode_probe<<<1, 256, smem>>>(dA, dP, dD, cb[0], cb[1], 2 * 128 * 128);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(pass ? D2.data() : D.data(), dD, 65536, cudaMemcpyDeviceToHost));
    }
    printf("lbo=%u sbo=%u: physical float index read for B(n, k), rows k=0..7, cols n=0..11\n", cb[0], cb[1]);
    for (int k = 0; k < 8; ++k) {
      for (int n = 0; n < 12; ++n) printf("%6d", (int)D2[k * 128 + n] * 1024 + (int)D[k * 128 + n]);
      printf("   ... n=32:%d n=127:%d\n", (int)D2[k * 128 + 32] * 1024 + (int)D[k * 128 + 32], (int)D2[k * 128 + 127] * 1024 + (int)D[k * 128 + 127]);
    }
  }
  return 0;
}
#else
int main() {
  const size_t smem = 3 * 128 * 128 * 4;
  CK(cudaFuncSetAttribute(gemm_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(rate_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  std::vector<float> A(128 * 128), B(128 * 128), D(128 * 128);
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (float)((s >> 8) & 0x3FF) / 512.0f - 1.0f; };  // tf32-exact
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, 65536)); CK(cudaMalloc(&dB, 65536)); CK(cudaMalloc(&dD, 65536));
  CK(cudaMemcpy(dA, A.data(), 65536, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), 65536, cudaMemcpyHostToDevice));
  const uint32_t cand[] = {128, 256, 512, 1024, 2048, 4096, 8192};
  for (uint32_t lb : cand) for (uint32_t sb : cand) {
    CK(cudaMemcpyToSymbol(MN_LBO, &lb, 4)); CK(cudaMemcpyToSymbol(MN_SBO, &sb, 4));
  for (int ts = 0; ts < 1; ++ts)
    for (int amn = 0; amn < 2; ++amn)
      for (int bmn = 0; bmn < 2; ++bmn) {
        if (ts && amn) continue;
        if (!amn && !bmn) continue;
        gemm_probe<<<1, 256, smem>>>(dA, dB, dD, amn, bmn, ts);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(D.data(), dD, 65536, cudaMemcpyDeviceToHost));
        double err = 0;
        for (int m = 0; m < 128; ++m)
          for (int n = 0; n < 128; ++n) {
            double ref = 0;
            for (int k = 0; k < 128; ++k) ref += (double)A[m * 128 + k] * B[n * 128 + k];
            err = fmax(err, fabs(ref - D[m * 128 + n]));
          }
        if (err < 1e-3) printf("view ts=%d amn=%d bmn=%d lbo=%u sbo=%u maxerr=%.3g\n", ts, amn, bmn, lb, sb, err);
      }
  }
  { uint32_t lb = R8 * 16, sb = C4 * 16; CK(cudaMemcpyToSymbol(MN_LBO, &lb, 4)); CK(cudaMemcpyToSymbol(MN_SBO, &sb, 4)); }
  // conversion: A = raw fp32 with low bits, B = identity -> D[m][n] = conv(A[m][n])
  for (int i = 0; i < 128 * 128; ++i) {
    s = s * 1664525u + 1013904223u;
    A[i] = 1.0f + (float)(s >> 9) / 8388608.0f;
    B[i] = (i / 128 == i % 128) ? 1.f : 0.f;
  }
  CK(cudaMemcpy(dA, A.data(), 65536, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), 65536, cudaMemcpyHostToDevice));
  for (int ts = 0; ts < 2; ++ts) {
    gemm_probe<<<1, 256, smem>>>(dA, dB, dD, 0, 0, ts);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, 65536, cudaMemcpyDeviceToHost));
    int ntr = 0, nrn = 0, nex = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 128; ++n) {
        const float a = A[m * 128 + n], d = D[m * 128 + n];
        ntr += d == tf32_trunc(a); nrn += d == tf32_rna(a); nex += d == a;
      }
    printf("conversion ts=%d: trunc-match %d rna-match %d exact %d of 16384\n", ts, ntr, nrn, nex);
  }
  long long* dc;
  CK(cudaMalloc(&dc, 8 * 148));
  const int Ns[] = {16, 32, 64, 128, 256};
  for (int ts = 0; ts < 2; ++ts)
    for (int v = 0; v < 3; ++v)
      for (int N : Ns) {
        const int amn = v == 1 || v == 2, bmn = v == 2;
        if (ts && amn) continue;
        const int iters = 200;
        rate_probe<<<148, 128, smem>>>(N, iters, amn, bmn, ts, dc, 1);
        CK(cudaDeviceSynchronize());
        long long c[148];
        CK(cudaMemcpy(c, dc, 8 * 148, cudaMemcpyDeviceToHost));
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
        const double per = (double)mx / (iters * 16);
        printf("rate ts=%d amn=%d bmn=%d N=%3d: %.1f cyc/MMA (floor %d), %.0f MAC/cyc/SM\n", ts, amn, bmn, N, per,
               128 * N / 256, 128.0 * N * 8 / per);
      }
  CK(cudaFuncSetAttribute(rate_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int N : {16, 32, 64, 128, 256}) {
      rate_warp<<<148, 128, smem>>>(N, 200, dc);
      CK(cudaDeviceSynchronize());
      long long c[148];
      CK(cudaMemcpy(c, dc, 8 * 148, cudaMemcpyDeviceToHost));
      long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
      printf("rate_warp N=%3d: %.1f cyc/MMA (floor %d)\n", N, (double)mx / (200 * 16), N / 2);
  }
  for (int ndst : {2, 4})
    for (int N : {16, 32, 64, 128}) {
      if (N * ndst > 512) continue;
      rate_probe<<<148, 128, smem>>>(N, 200, 0, 0, 0, dc, ndst);
      CK(cudaDeviceSynchronize());
      long long c[148];
      CK(cudaMemcpy(c, dc, 8 * 148, cudaMemcpyDeviceToHost));
      long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
      printf("rate ndst=%d N=%3d: %.1f cyc/MMA\n", ndst, N, (double)mx / (200 * 16));
    }
  return 0;
}
#endif
