// mbar_cost.cu -- single-thread cost of mbarrier / bulk-copy primitives (cycles per op, 64-op loops).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
extern __shared__ __align__(1024) uint8_t dsm[];
__global__ void k(const uint8_t* src, long long* out) {
  __shared__ uint64_t bars[70];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 70; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(&bars[i])), "r"((1 << 20) - 1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long t0, t1;
  uint32_t b0 = su32(&bars[0]);
  // A: plain arrive (count never reached)
  t0 = clock64();
  for (int i = 0; i < 64; i++) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(b0) : "memory");
  t1 = clock64(); out[0] = (t1 - t0) / 64;
  // B: test_wait on a phase that is complete (parity 1 of a fresh barrier = previous phase, complete)
  t0 = clock64();
  uint32_t acc = 0;
  for (int i = 0; i < 64; i++) {
    uint32_t ok;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(su32(&bars[1])) : "memory");
    acc += ok;
  }
  t1 = clock64(); out[1] = (t1 - t0) / 64; out[9] = acc;
  // C: arrive.expect_tx (no copy) on distinct barriers
  t0 = clock64();
  for (int i = 0; i < 32; i++) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&bars[2 + i])), "r"(4096) : "memory");
  t1 = clock64(); out[2] = (t1 - t0) / 32;
  // D: bulk copies of 4 KB onto those barriers (completing their tx), no waits
  t0 = clock64();
  for (int i = 0; i < 32; i++)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(su32(dsm) + (i & 31) * 4096), "l"(src + i * 4096), "r"(4096), "r"(su32(&bars[2 + i])) : "memory");
  t1 = clock64(); out[3] = (t1 - t0) / 32;
  // E: 1 KB copies
  for (int i = 0; i < 32; i++) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&bars[34 + i])), "r"(1024) : "memory");
  t0 = clock64();
  for (int i = 0; i < 32; i++)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(su32(dsm) + (i & 31) * 4096), "l"(src + i * 4096), "r"(1024), "r"(su32(&bars[34 + i])) : "memory");
  t1 = clock64(); out[4] = (t1 - t0) / 32;
}
int main() {
  uint8_t* src; cudaMalloc(&src, 1 << 22); cudaMemset(src, 0, 1 << 22);
  long long* d; cudaMalloc(&d, 16 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  k<<<1, 32, 132 * 1024>>>(src, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[16]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("arrive %lld | try_wait(done) %lld | arrive.expect_tx %lld | bulk 4KB issue %lld | bulk 1KB issue %lld cycles/op (%s)\n",
         h[0], h[1], h[2], h[3], h[4], cudaGetErrorString(e));
  return 0;
}
