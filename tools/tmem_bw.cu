// tmem_bw.cu -- microbenchmark: tcgen05.ld (32x32b.xN) throughput per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_bw tools/tmem_bw.cu && /tmp/tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int X>
__global__ void k(int iters, unsigned long long* cycles, uint32_t* sink, int nwarps) {
  __shared__ uint32_t slot;
  int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  unsigned long long t0 = clock64();
  if (warp < nwarps) {
    for (int it = 0; it < iters; it++) {
      for (int c = 0; c < 512; c += 16 * X) {
        uint32_t r[16 * X];
        if constexpr (X == 1) {
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]) : "r"(base + c));
        } else {
          #pragma unroll
          for (int q = 0; q < X; q++)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(r[16*q+0]),"=r"(r[16*q+1]),"=r"(r[16*q+2]),"=r"(r[16*q+3]),"=r"(r[16*q+4]),"=r"(r[16*q+5]),"=r"(r[16*q+6]),"=r"(r[16*q+7]),"=r"(r[16*q+8]),"=r"(r[16*q+9]),"=r"(r[16*q+10]),"=r"(r[16*q+11]),"=r"(r[16*q+12]),"=r"(r[16*q+13]),"=r"(r[16*q+14]),"=r"(r[16*q+15]) : "r"(base + c + 16*q));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        #pragma unroll
        for (int j = 0; j < 16 * X; j++) acc += r[j];
      }
    }
  }
  unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(slot), "r"(512));
}
int main() {
  unsigned long long* cyc; uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8); cudaMalloc(&sink, 148 * 1024 * 4);
  int iters = 200;
  for (int nw : {4, 8, 16}) {
    for (int x : {1, 2, 4}) {
      if (x == 1) k<1><<<148, nw * 32>>>(iters, cyc, sink, nw);
      if (x == 2) k<2><<<148, nw * 32>>>(iters, cyc, sink, nw);
      if (x == 4) k<4><<<148, nw * 32>>>(iters, cyc, sink, nw);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double bytes = (double)iters * 512 * 128 * 4 * (nw / 4);   // each quadrant's warps read all 512 cols
      printf("warps %2d  ld x16 * %d in flight: %.1f bytes/cycle/SM  (%s)\n", nw, x, bytes / h[0], cudaGetErrorString(e));
    }
  }
  return 0;
}
