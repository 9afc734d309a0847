// umma_rate.cu -- kind::i8 UMMA (SS, K-major no-swizzle) issue-to-completion cost vs N and M, single
// issuing thread, 256 back-to-back UMMAs then one commit.  Also: the same with 4 UMMAs per distinct
// A/B descriptor pair rotating over 4 smem stages.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}
extern __shared__ __align__(1024) uint8_t dsm[];
__global__ void k(int M, int N, int nmma, int reps, long long* out, int variant) {
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 65536; i += blockDim.x) dsm[i] = (uint8_t)i;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = slot;
  if (threadIdx.x == 0) {
    uint32_t id = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    uint32_t B = su32(&bar);
    long long best = 1ll << 60;
    for (int r = 0; r < reps; r++) {
      long long t0 = clock64();
      if (variant == 1) {   // constant descriptors, unrolled by 8, alternating two accumulators
        uint32_t a = su32(dsm), b = su32(dsm) + 32768;
        const uint64_t ad = (uint64_t)((a & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
        const uint64_t bd = (uint64_t)((b & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
        for (int m = 0; m < nmma; m += 8) {
#pragma unroll
          for (int q = 0; q < 8; q++)
            asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;"
                         :: "r"(tm + (uint32_t)((q & 1) * 256)), "l"(ad), "l"(bd), "r"(id) : "memory");
        }
      } else if (variant == 2) {   // constant descriptors, distinct accumulators per MMA (8 x N cols)
        uint32_t a = su32(dsm), b = su32(dsm) + 32768;
        const uint64_t ad = (uint64_t)((a & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
        const uint64_t bd = (uint64_t)((b & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
        for (int m = 0; m < nmma; m += 8) {
#pragma unroll
          for (int q = 0; q < 8; q++)
            asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;"
                         :: "r"(tm + (uint32_t)(q * (N < 64 ? N : 64))), "l"(ad), "l"(bd), "r"(id) : "memory");
        }
      } else
      for (int m = 0; m < nmma; m++) {
        uint32_t a = su32(dsm) + (m & 3) * 8192, b = su32(dsm) + 32768 + (m & 3) * 8192;
        uint64_t ad = (uint64_t)((a & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
        uint64_t bd = (uint64_t)((b & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
                     :: "r"(tm + (uint32_t)((m & 1) * 256)), "l"(ad), "l"(bd), "r"(id), "r"(m) : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(B) : "memory");
      while (!try_wait(B, r & 1)) {}
      long long t1 = clock64();
      if (t1 - t0 < best) best = t1 - t0;
    }
    out[0] = best;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tm), "r"(512));
}
int main() {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int v : {0, 1, 2})
  for (int M : {128})
    for (int N : {16, 32, 64, 128, 256}) {
      k<<<1, 128, 65536>>>(M, N, 256, 5, d, v);
      cudaError_t e = cudaDeviceSynchronize();
      long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      double per = (h - 400) / 256.0;
      printf("variant %d M=%3d N=%3d: %7.1f cycles/UMMA  %7.0f int8 MAC/cycle  (%s)\n", v, M, N, per, M * N * 32 / per, cudaGetErrorString(e));
    }
  return 0;
}
