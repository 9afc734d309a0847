// commit_tput.cu -- THROUGHPUT of back-to-back tcgen05.commit (each to its own mbarrier, the issuing
// thread does not wait in between; the burst is timed to its last commit), with 0 / 1 / 2 / 4 UMMAs (M=128, N=16 or 64, K=32, kind::i8) before
// each commit; plus the per-commit completion times of one burst.  Single CTA, single issuing thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ct tools/commit_tput.cu && /tmp/ct
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}
constexpr int kBars = 16;
__global__ void k(int nmma, int n_n, int bursts, long long* out) {
  __shared__ __align__(1024) uint8_t sm[8192 + 1024];
  __shared__ uint64_t bar[kBars];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 9216; i += blockDim.x) sm[i] = 0;
  if (threadIdx.x == 0) {
    for (int b = 0; b < kBars; b++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = su32(sm), b = su32(sm + 4096);
    const uint64_t ad = (uint64_t)((a & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
    const uint64_t bd = (uint64_t)((b & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
    const uint32_t id = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n_n >> 3) << 17) | ((128 >> 4) << 24);
    long long done[kBars];
    long long t0 = clock64();
    for (int r = 0; r < bursts; r++) {
      for (int i = 0; i < kBars; i++) {
        for (int m = 0; m < nmma; m++)
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
                       ::"r"(tm), "l"(ad), "l"(bd), "r"(id), "r"(m) : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(su32(&bar[i])) : "memory");
      }
      // wait for the LAST commit only (commits complete in issue order), then retire the others
      while (!try_wait(su32(&bar[kBars - 1]), r & 1)) {}
      if (r == bursts - 1) done[kBars - 1] = clock64();
      for (int i = 0; i < kBars - 1; i++) {
        const bool ok = try_wait(su32(&bar[i]), r & 1);
        if (r == bursts - 1) done[i] = ok ? 1 : 0;   // 1: already complete when the last one was
        while (!try_wait(su32(&bar[i]), r & 1)) {}
      }
    }
    long long t1 = clock64();
    out[0] = (t1 - t0) / ((long long)bursts * kBars);
    for (int i = 0; i < kBars - 1; i++) out[1 + i] = done[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(128));
}
int main() {
  long long* d;
  cudaMalloc(&d, 8 * (1 + kBars));
  struct { int nmma, n; } cases[] = {{0, 16}, {1, 16}, {2, 16}, {4, 16}, {1, 64}, {2, 64}, {4, 64}};
  for (auto& c : cases) {
    k<<<1, 128>>>(c.nmma, c.n, 200, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[1 + kBars];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int early = 0;
    for (int i = 1; i < kBars; i++) early += (int)h[i];
    printf("%d UMMA (N=%2d) + commit, bursts of 16: %5lld cycles per commit; %d/15 earlier commits complete with the last",
           c.nmma, c.n, h[0], early);
    printf("  (%s)\n", cudaGetErrorString(e));
  }
  return 0;
}
