// bulk_bw.cu -- cp.async.bulk (1-D TMA) global->shared streaming throughput per SM and chip-wide,
// vs copy size and ring depth; consumer = one thread waiting on full barriers and re-arming.
// share > 1: groups of `share` consecutive CTAs read the same addresses (L2 reuse pattern).
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
__global__ void k(const uint8_t* src, long long bytes_per_cta, int copy, int depth, int share, long long* cyc, int nprod) {
  __shared__ uint64_t bars[32];
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int w = threadIdx.x / 32;
  if ((threadIdx.x & 31) != 0 || w >= nprod) return;
  const uint8_t* base = src + (long long)(blockIdx.x / share) * bytes_per_cta;
  long long n = bytes_per_cta / copy;
  long long t0 = clock64();
  // producer w owns stages s with s % nprod == w (and the copies landing in them)
  for (long long i = 0; i < n + depth; i++) {
    if ((i % depth) % nprod != w) continue;
    if (i >= depth) {   // consume copy i - depth
      long long j = i - depth;
      int s = j % depth;
      while (!try_wait(su32(&bars[s]), (j / depth) & 1)) {}
    }
    if (i < n) {
      int s = i % depth;
      uint32_t bar = su32(&bars[s]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(copy) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(su32(dsm) + s * copy), "l"(base + i * copy), "r"(copy), "r"(bar) : "memory");
    }
  }
  if (w == 0) cyc[blockIdx.x] = clock64() - t0;
}
int main() {
  const long long per = 8ll << 20;   // 8 MB per CTA
  uint8_t* src; cudaMalloc(&src, 148 * per);
  cudaMemset(src, 1, 148 * per);
  long long* cyc; cudaMalloc(&cyc, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct C { int copy, depth, share; };
  C cs[] = {{4096, 32, 4}, {16384, 12, 4}, {32768, 6, 4}, {4096, 32, 1}, {16384, 12, 1}};
  for (int np : {1, 2, 4})
  for (auto c : cs) {
    int smem = c.copy * c.depth;
    k<<<148, 128, smem>>>(src, per, c.copy, c.depth, c.share, cyc, np);   // warm
    cudaEventRecord(e0);
    k<<<148, 128, smem>>>(src, per, c.copy, c.depth, c.share, cyc, np);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double bpc = (double)per / h[0];
    printf("nprod %d copy %6d depth %2d share %d: %7.1f B/cyc/SM  chip %7.1f GB/s  unique-from-L2/DRAM %7.1f GB/s (%s)\n",
           np, c.copy, c.depth, c.share, bpc, 148.0 * per / (ms * 1e6), 148.0 * per / c.share / (ms * 1e6), cudaGetErrorString(err));
  }
  return 0;
}
