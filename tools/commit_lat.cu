// commit_lat.cu -- latency of tcgen05.commit -> mbarrier (with 0 / 1 / 8 UMMAs in flight), and of a
// plain mbarrier arrive -> wait, single thread.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cl tools/commit_lat.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}
__global__ void k(int mode, int nmma, int iters, long long* out) {
  __shared__ __align__(1024) uint8_t sm[8192 + 1024];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(su32(&slot)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 9216; i += blockDim.x) sm[i] = 0;
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
    uint32_t a = su32(sm), b = su32(sm + 4096);
    uint64_t ad = (uint64_t)((a & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
    uint64_t bd = (uint64_t)((b & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
    uint32_t id = (2u << 4) | (1u << 7) | (1u << 10) | ((16 >> 3) << 17) | ((128 >> 4) << 24);
    uint32_t B = su32(&bar);
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
      if (mode == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(B) : "memory");
      } else {
        for (int m = 0; m < nmma; m++)
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
                       :: "r"(tm), "l"(ad), "l"(bd), "r"(id), "r"(m) : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(B) : "memory");
      }
      while (!try_wait(B, it & 1)) {}
    }
    long long t1 = clock64();
    out[0] = (t1 - t0) / iters;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tm), "r"(64));
}
int main() {
  long long* d; cudaMalloc(&d, 8);
  struct { int mode, nmma; const char* name; } cases[] = {{0, 0, "mbarrier.arrive -> wait"}, {1, 0, "commit (no MMA) -> wait"},
    {1, 1, "1 UMMA 128x16x32 + commit -> wait"}, {1, 8, "8 UMMA + commit -> wait"}, {1, 32, "32 UMMA + commit -> wait"}};
  for (auto& c : cases) {
    k<<<1, 128>>>(c.mode, c.nmma, 2000, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %6lld cycles/iter  (%s)\n", c.name, h, cudaGetErrorString(e));
  }
  return 0;
}
