// copy_lat.cu -- are 1-D bulk copies (cp.async.bulk) pipelined?  One thread issues N copies of S bytes up
// front (distinct mbarriers), then waits for all: time vs N and S.  Compared with the same bytes moved by
// 4 warps of cp.async (LDGSTS, 16 B per thread).  148 CTAs, each its own 4 MB region (DRAM) or all the
// same region (L2).
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
__global__ void k(const uint8_t* src, int n, int size, int mode, int same, long long* cyc) {
  __shared__ uint64_t bars[64];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 64; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const uint8_t* base = src + (same ? 0 : (long long)blockIdx.x * (4 << 20));
  long long t0 = clock64();
  if (mode == 0) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < n; i++) {
        uint32_t bar = su32(&bars[i]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(size) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(su32(dsm) + (uint32_t)((long long)i * size % (192 * 1024))), "l"(base + (long long)i * size), "r"(size), "r"(bar) : "memory");
      }
      for (int i = 0; i < n; i++) while (!try_wait(su32(&bars[i]), 0)) {}
    }
  } else {
    // 128 threads, 16 B each per instruction
    long long total = (long long)n * size;
    for (long long off = threadIdx.x * 16; off < total; off += 128 * 16) {
      uint32_t d = su32(dsm) + (uint32_t)(off % (192 * 1024));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(d), "l"(base + off) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}
int main() {
  uint8_t* src; cudaMalloc(&src, 148ll * (4 << 20)); cudaMemset(src, 1, 148ll * (4 << 20));
  long long* cyc; cudaMalloc(&cyc, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * 1024);
  for (int same : {0, 1})
    for (int mode : {0, 1})
      for (int size : {4096, 16384, 32768})
        for (int n : {1, 8, 32}) {
          if ((long long)n * size > (4 << 20)) continue;
          k<<<148, 128, 192 * 1024>>>(src, n, size, mode, same, cyc);
          k<<<148, 128, 192 * 1024>>>(src, n, size, mode, same, cyc);
          cudaError_t e = cudaDeviceSynchronize();
          long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
          long long mx = 0; double avg = 0;
          for (int i = 0; i < 148; i++) { mx = h[i] > mx ? h[i] : mx; avg += h[i] / 148.0; }
          printf("%s %s size %6d n %2d: avg %8.0f cyc (%6.0f per copy, %5.1f B/cyc/SM)  max %8lld (%s)\n",
                 same ? "L2  " : "DRAM", mode ? "ldgsts" : "bulk  ", size, n, avg, avg / n, (double)n * size / avg, mx,
                 cudaGetErrorString(e));
        }
  return 0;
}
