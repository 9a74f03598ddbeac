// Standalone probe (sm_100a): tcgen05 kind::tf32 with BOTH operands MN-major
// in the SWIZZLE_128B_BASE32B layout (layout type 1), the layout GEMM3 of the
// TransR step reads its row-major U / DZ tiles in (K = rows, MN = features).
//   D[i][j] = sum_k A[k][i] * B[k][j],  A, B: K x 128 row tiles
// Byte offset of (k, mn): (mn / 32) * LBO + k * 128 + ((((mn % 32) / 8) ^ (k & 3)) * 32) + (mn % 8) * 4
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_mn_probe tools/umma_mn_probe.cu && ./umma_mn_probe
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

constexpr int K = 32;  // rows per tile in the probe (4 MMAs of K = 8)

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc_sw128_32b(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (1ull << 61);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int amn, int bmn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amn << 15) | ((uint32_t)bmn << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__host__ __device__ inline int off_bytes(int k, int mn, int lbo) {
  return (mn / 32) * lbo + k * 128 + ((((mn % 32) / 8) ^ (k & 3)) * 32) + (mn % 8) * 4;
}

__global__ void probe(const float* A, const float* B, float* D, int lbo_mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int lbo = K * 128;  // MN blocks of 32 follow each other after K rows
  uint8_t* As = sm;
  uint8_t* Bs = sm + 4 * lbo;
  for (int i = threadIdx.x; i < K * 128; i += blockDim.x) {
    const int k = i / 128, mn = i % 128;
    *reinterpret_cast<float*>(As + off_bytes(k, mn, lbo)) = A[i];
    *reinterpret_cast<float*>(Bs + off_bytes(k, mn, lbo)) = B[i];
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tbase)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = tbase;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_tf32(128, 128, 1, 1);
    for (int s = 0; s < K / 8; ++s) {
      const uint64_t ad = desc_sw128_32b(su32(As) + s * 1024, lbo_mode ? lbo : 512, lbo_mode ? 512 : lbo);
      const uint64_t bd = desc_sw128_32b(su32(Bs) + s * 1024, lbo_mode ? lbo : 512, lbo_mode ? 512 : lbo);
      const uint32_t acc = s > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                   ::"r"(t), "l"(ad), "l"(bd), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred d;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 d, [%0], 0;\n\t@!d bra W_%=;\n\t}\n" ::"r"(su32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int w = threadIdx.x >> 5;
  if (w < 4) {
    for (int c = 0; c < 128; c += 16) {
      uint32_t r[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
                     "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                   : "r"(t + ((uint32_t)(w * 32) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int q = 0; q < 16; ++q) D[threadIdx.x * 128 + c + q] = __uint_as_float(r[q]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(t) : "memory");
}

int main() {
  std::vector<float> A(K * 128), B(K * 128), D(128 * 128);
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; float x = ((s >> 8) & 0xFFFF) / 65536.0f - 0.5f;
                     uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; memcpy(&x, &u, 4); return x; };
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  const int smem = 2 * 4 * K * 128 + 1024;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int mode = 0; mode < 2; ++mode) {
    CK(cudaMemset(dD, 0, D.size() * 4));
    probe<<<1, 128, smem>>>(dA, dB, dD, mode);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0;
    for (int i = 0; i < 128; ++i)
      for (int j = 0; j < 128; ++j) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)A[k * 128 + i] * B[k * 128 + j];
        maxerr = fmax(maxerr, fabs(ref - D[i * 128 + j]));
      }
    printf("mode %s: max |D - ref| = %.3g (D[0][0]=%g)\n", mode ? "LBO=MN-block,SBO=K-group" : "LBO=K-group,SBO=MN-block",
           maxerr, D[0]);
  }
  return 0;
}
