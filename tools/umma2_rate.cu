// umma2_rate.cu -- issue rate of back-to-back tcgen05.mma.kind::i8 (K = 32, N = 128) on one CTA (M = 128,
// cta_group::1) vs a CTA pair (M = 256, cta_group::2): cycles per UMMA on the issuing SM's clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma2_rate umma2_rate.cu && ./umma2_rate
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cta_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void wait_parity(uint32_t bar, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                 : "=r"(ok) : "r"(bar), "r"(par) : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}

template <int PAIR>
__global__ void rate(int iters, int N, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const uint32_t rank = PAIR ? cta_rank() : 0;
  if (threadIdx.x < 32) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base)), "r"(256));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base)), "r"(256));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  for (int i = threadIdx.x * 16; i < 64 * 1024; i += blockDim.x * 16) *(int4*)(smem + i) = make_int4(1, 2, 3, 4);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (PAIR) cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tmem_base;
  const uint32_t M = PAIR ? 256 : 128;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((M >> 4) << 24);
  if (rank == 0 && threadIdx.x == 0) {
    const uint64_t ad = desc(smem_u32(smem)), bd = desc(smem_u32(smem) + 16384);
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
      if (PAIR)
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p; }"
                     :: "r"(tb), "l"(ad), "l"(bd), "r"(idesc), "r"(1));
      else
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
                     :: "r"(tb), "l"(ad), "l"(bd), "r"(idesc), "r"(1));
    }
    if (PAIR)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   :: "r"(smem_u32(&bar)), "h"((uint16_t)3));
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
    wait_parity(smem_u32(&bar), 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  if (PAIR && rank == 1 && threadIdx.x == 0) wait_parity(smem_u32(&bar), 0);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (PAIR) cluster_sync();
  if (threadIdx.x < 32) {
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tb), "r"(256));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tb), "r"(256));
  }
}

int main() {
  long long* d; cudaMalloc(&d, 16 * sizeof(long long));
  const int iters = 4096;
  cudaFuncSetAttribute(rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int N : {64, 128, 256}) {
    long long h[2];
    rate<0><<<1, 128, 64 * 1024>>>(iters, N, d);
    cudaDeviceSynchronize(); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    const double c1 = (double)h[0] / iters;
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(2); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 64 * 1024;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, rate<1>, iters, N, d);
    cudaError_t e = cudaDeviceSynchronize(); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    const double c2 = (double)h[0] / iters;
    printf("N=%d: cta_group::1 M=128 %.1f cycles/UMMA (%.0f MAC/cycle/SM); cta_group::2 M=256 %.1f cycles/UMMA (%.0f MAC/cycle/SM) %s\n",
           N, c1, 128.0 * N * 32 / c1, c2, 128.0 * N * 32 / c2, cudaGetErrorString(e));
  }
  return 0;
}
